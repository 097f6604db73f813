# 4 GPUs: multi-GPU tests, NVLink peaks, NEXT-3 crossover, bench lines, pack-stream A/B, P=8-settings stress
N=4
O=gpurun_out/r02/p4; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log
tail -2 $O/pytest_multi.log
timeout 400 $T --master-port 29511 scripts/nvlink_peaks.py $O/nvlink_peaks.json > $O/nvlink.log 2>&1; echo "nvl rc=$?" >> $O/nvlink.log
timeout 600 $T --master-port 29512 scripts/scheme_crossover.py $O/scheme_crossover.json > $O/crossover.log 2>&1; echo "xover rc=$?" >> $O/crossover.log
tail -2 $O/nvlink.log $O/crossover.log
port=29520
run() { name=$1; shift; port=$((port+1)); timeout 300 env "$@" $T --master-port $port bench.py --gpus $N --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['step']['frac_pipelined'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"; }
for cfg in c3 c1 c2 c4; do
  ARGS="--config $cfg" run bench_$cfg POS_PACK_STREAM=0
  ARGS="--config $cfg" run pk_$cfg POS_PACK_STREAM=1
done
ARGS="--config c1" run c1_pair512 POS_SFB_PAIR_KP=512
ARGS="--config c4 --bucket-mb 64" run c4_b64 POS_PACK_STREAM=0
for i in 1 2 3; do
  ARGS="--config c3" run stress_c3_$i POS_NVLS_CTAS=16 POS_SFB_PAIR=1
  ARGS="--config c1" run stress_c1_$i POS_NVLS_CTAS=16 POS_SFB_PAIR=1
done
