# N GPUs: flag-mode packs on their own stream (POS_PACK_STREAM=1) vs on the comm stream, 4 configs x 2
O=gpurun_out/r02/pk; mkdir -p $O
export POS_TIMEOUT_MS=20000
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
port=29350
for rep in 1 2; do
for cfg in c3 c2 c1 c4; do
  for p in 1 0; do
    port=$((port+1))
    timeout 300 env POS_PACK_STREAM=$p $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_pk${p}_n${NG}_$rep.json 2> $O/b_${cfg}_pk${p}_n${NG}_$rep.err
    echo "$cfg pk=$p rc=$? $(python -c "import json; d=json.loads(open('$O/b_${cfg}_pk${p}_n${NG}_$rep.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))" 2>&1 | tail -1)"
  done
done
done
