# 2 GPUs: PS bucket size at P = 2 on the final defaults (32 MiB vs the 64 MiB default)
O=gpurun_out/r02/bucket; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=28700
for cfg in c2 c4 c3; do port=$((port+1))
  timeout 300 $T --master-port $port bench.py --gpus 2 --config $cfg --bucket-mb 32 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_32.json 2> $O/b_${cfg}_32.err
  echo "$cfg 32MiB rc=$? $(python -c "import json; d=json.loads(open('$O/b_${cfg}_32.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))" 2>&1 | tail -1)"
done
