# 4 GPUs: NVLS PS grid sweep for VGG19-22K / VGG19
O=gpurun_out/r02/p4ctas; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30010
for cfg in c3 c2; do for c in 24 32 48 64 96; do port=$((port+1))
  POS_NVLS_CTAS=$c timeout 300 $T --master-port $port bench.py --gpus 4 --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/${cfg}_c$c.json 2>/dev/null
  echo "$cfg ctas=$c $(python -c "import json; d=json.loads(open('$O/${cfg}_c$c.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), d['trace_timeline_us'])" 2>&1 | tail -1)"
done; done
