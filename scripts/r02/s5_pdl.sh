# 4 GPUs: programmatic dependent launch between consecutive fused PS kernels (explicit trigger after
# the epoch release): multi-GPU tests with POS_PS_PDL=1, then A/B at P = 4 and P = 2
O=gpurun_out/r02/pdl2; mkdir -p $O
export POS_TIMEOUT_MS=20000
POS_PS_PDL=1 timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi_p4.log 2>&1; echo "multi rc=$?"; tail -1 $O/pytest_multi_p4.log
port=29250
for NG in 4 2; do
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
for cfg in c3 c2 c4 c1; do
  for p in 1 0; do
    port=$((port+1))
    timeout 300 env POS_PS_PDL=$p $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_p${p}_n${NG}.json 2> $O/b_${cfg}_p${p}_n${NG}.err
    echo "P$NG $cfg pdl=$p rc=$? $(python -c "
import json; d=json.loads(open('$O/b_${cfg}_p${p}_n${NG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), [(r[0][:12], r[2], r[3]) for r in sorted(d['trace_timeline_us'], key=lambda r: r[2]) if r[1]=='PS'])" 2>&1 | tail -1)"
  done
done
done
