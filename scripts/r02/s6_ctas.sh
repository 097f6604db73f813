# 2 GPUs: PS grid (POS_NVLS_CTAS) at P = 2 on the final defaults
O=gpurun_out/r02/ctas; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=28950
for cfg in c3 c2; do for n in 96 128 64; do port=$((port+1))
  timeout 300 env POS_NVLS_CTAS=$n $T --master-port $port bench.py --gpus 2 --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_${n}.json 2> $O/b_${cfg}_${n}.err
  echo "$cfg ctas=$n rc=$? $(python -c "import json; d=json.loads(open('$O/b_${cfg}_${n}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))" 2>&1 | tail -1)"
done; done
