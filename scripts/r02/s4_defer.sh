# N GPUs: deferred PS exit barrier (epoch-slot barriers): multi-GPU tests, then A/B bench lines
# (POS_PS_DEFER=1 new default vs 0)
O=gpurun_out/r02/defer; mkdir -p $O
export POS_TIMEOUT_MS=20000
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi_$NG.log 2>&1; echo "multi rc=$?"; tail -2 $O/pytest_multi_$NG.log | cut -c1-800
port=29600
for rep in 1 2; do
for cfg in c3 c2 c1 c4; do
  for d in 1 0; do
    port=$((port+1))
    timeout 300 env POS_PS_DEFER=$d $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_d${d}_n${NG}_$rep.json 2> $O/b_${cfg}_d${d}_n${NG}_$rep.err
    echo "$cfg defer=$d rc=$? $(python -c "import json; d=json.loads(open('$O/b_${cfg}_d${d}_n${NG}_$rep.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(d['roofline']['step']['frac_pipelined'],3))" 2>&1 | tail -1)"
  done
done
done
