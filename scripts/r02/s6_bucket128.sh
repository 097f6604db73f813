# 2 GPUs: one 80 MB PS unit (128 MiB buckets) at P = 2 vs the 64 MiB default (two units)
O=gpurun_out/r02/bucket; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=28500
for cfg in c3 c2; do port=$((port+1))
  timeout 200 $T --master-port $port bench.py --gpus 2 --config $cfg --bucket-mb 128 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_128.json 2> $O/b_${cfg}_128.err
  echo "$cfg 128MiB rc=$? $(python -c "import json; d=json.loads(open('$O/b_${cfg}_128.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), d['config']['ps_units'])" 2>&1 | tail -1)"
done
