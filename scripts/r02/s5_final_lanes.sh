# 4 GPUs: lane count decided by the scheduler (two lanes when the PS units dominate): multi-GPU tests
# at P = 4, default bench lines at P = 4 (all configs) and P = 2 (Inception-V3)
O=gpurun_out/r02/final7; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi_p4.log 2>&1; echo "multi p4 rc=$?"; tail -1 $O/pytest_multi_p4.log
port=29050
for run in "4 c4" "4 c2" "4 c3" "4 c1" "2 c4"; do set -- $run; N=$1; cfg=$2; port=$((port+1))
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  timeout 400 $T --master-port $port bench.py --gpus $N --config $cfg > $O/bench_${cfg}_n$N.json 2> $O/bench_${cfg}_n$N.err
  echo "P$N $cfg rc=$? $(python -c "import json; d=json.loads(open('$O/bench_${cfg}_n$N.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(r['step']['frac_pipelined'],3), d['e2e'] and round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
