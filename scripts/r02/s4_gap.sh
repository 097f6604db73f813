# N GPUs: PS-unit launch gaps next to the reconstructions: reconstruction grid cap (POS_SFB_MAX_CTAS)
O=gpurun_out/r02/gap; mkdir -p $O
export POS_TIMEOUT_MS=20000
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
port=29650
for cfg in c3 c2; do
  for m in 0 140 128; do
    port=$((port+1))
    timeout 300 env POS_SFB_MAX_CTAS=$m $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_m${m}_n${NG}.json 2> $O/b_${cfg}_m${m}_n${NG}.err
    echo "$cfg max_ctas=$m rc=$? $(python -c "
import json; d=json.loads(open('$O/b_${cfg}_m${m}_n${NG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))
for r in sorted(d['trace_timeline_us'], key=lambda r: r[2]): print('   ', r)" 2>&1 | tail -12)"
  done
done
