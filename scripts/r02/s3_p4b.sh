# 4 GPUs with the round-2 defaults: multi-GPU tests, bench lines, bucket / reduce-order A/B, exposure at P=4
N=4
O=gpurun_out/r02/p4b; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log; tail -2 $O/pytest_multi.log
port=29860
run() { name=$1; shift; port=$((port+1)); timeout 300 env "$@" $T --master-port $port bench.py --gpus $N --steps 50 --warmup 10 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(d['roofline']['step']['frac_pipelined'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"; }
for cfg in c3 c1 c2 c4; do ARGS="--config $cfg --no-cpu-baseline" run bench_$cfg X=1; done
for cfg in c3 c2 c4; do
  ARGS="--config $cfg --bucket-mb 16 --no-cpu-baseline --no-e2e --no-tf32" run b16_$cfg X=1
  ARGS="--config $cfg --no-cpu-baseline --no-e2e --no-tf32" run ro_$cfg POS_REDUCE_ORDER=1
done
bash scripts/r02/s3_wfbp.sh 4
