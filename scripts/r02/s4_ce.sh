# 2 GPUs: copy-engine PS transport (POS_PS_CE=1): full-model oracle test incl. the CE context, then
# A/B bench lines (CE vs the fused SM kernel) on the four configs
O=gpurun_out/r02/ce; mkdir -p $O
export POS_TIMEOUT_MS=20000
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi_model.py -x -q -s > $O/pytest_mm_$NG.log 2>&1; echo "mm rc=$?"; tail -2 $O/pytest_mm_$NG.log | cut -c1-600
port=29700
for rep in 1 2; do
for cfg in c2 c3 c1 c4; do
  for ce in 1 0; do
    port=$((port+1))
    timeout 300 env POS_PS_CE=$ce $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_ce${ce}_n${NG}_$rep.json 2> $O/b_${cfg}_ce${ce}_n${NG}_$rep.err
    echo "$cfg ce=$ce rc=$? $(python -c "import json; d=json.loads(open('$O/b_${cfg}_ce${ce}_n${NG}_$rep.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(d['roofline']['step']['frac_pipelined'],3))" 2>&1 | tail -1)"
  done
done
done
