# 2 GPUs: multi-GPU tests (incl. two PS lanes), event-free timelines at P=2
O=gpurun_out/r02/p2tl; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log; tail -2 $O/pytest_multi.log
port=29950
run() { name=$1; shift; port=$((port+1)); timeout 300 env "$@" $T --master-port $port bench.py --gpus 2 --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(d['roofline']['step']['frac_pipelined'],3), d['trace_timeline_us'])" 2>&1 | tail -1)"; }
for cfg in c3 c2 c4 c1; do ARGS="--config $cfg" run def_$cfg X=1; done
ARGS="--config c2" run l2_c2 POS_PS_LANES=2
ARGS="--config c3" run l2_c3 POS_PS_LANES=2
ARGS="--config c2 --bucket-mb 16" run b16_c2 X=1
