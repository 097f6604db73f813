# 4 GPUs: scheduler-chosen lane count (threshold 0.5): Inception-V3 at P = 4 / 2 should take two lanes
O=gpurun_out/r02/final8; mkdir -p $O
export POS_TIMEOUT_MS=20000
port=29070
for run in "4 c4" "2 c4" "4 c2"; do set -- $run; N=$1; cfg=$2; port=$((port+1))
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  timeout 400 $T --master-port $port bench.py --gpus $N --config $cfg > $O/bench_${cfg}_n$N.json 2> $O/bench_${cfg}_n$N.err
  echo "P$N $cfg rc=$? $(python -c "import json; d=json.loads(open('$O/bench_${cfg}_n$N.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(r['step']['frac_pipelined'],3), d['e2e'] and round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'], [(x[0][:10], x[2], x[3]) for x in sorted(d['trace_timeline_us'], key=lambda x: x[2])][:4])" 2>&1 | tail -1)"
done
