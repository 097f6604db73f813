# N GPUs: programmatic dependent launch of the fused PS kernels (POS_PS_PDL=1 vs 0)
O=gpurun_out/r02/pdl; mkdir -p $O
export POS_TIMEOUT_MS=20000
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
port=29550
for cfg in c3 c2 c4; do
  for p in 1 0; do
    port=$((port+1))
    timeout 300 env POS_PS_PDL=$p $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_p${p}_n${NG}.json 2> $O/b_${cfg}_p${p}_n${NG}.err
    echo "$cfg pdl=$p rc=$? $(python -c "
import json; d=json.loads(open('$O/b_${cfg}_p${p}_n${NG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))
for r in sorted(d['trace_timeline_us'], key=lambda r: r[2]): print('   ', r)" 2>&1 | tail -9)"
  done
done
