# 2 GPUs: multi-GPU parity with the pack stream, bench lines (pack stream on / off), then the wide-tile A4 test on GPU 0
export POS_TIMEOUT_MS=20000
mkdir -p gpurun_out/r02/combo1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > gpurun_out/r02/combo1/pytest_multi.log 2>&1; echo "multi rc=$?" >> gpurun_out/r02/combo1/pytest_multi.log
tail -2 gpurun_out/r02/combo1/pytest_multi.log
bash scripts/r02/s3_pb.sh 2 pk
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for cfg in c3 c1; do POS_PACK_STREAM=0 timeout 300 $T --master-port $((29700 + ${#cfg} + RANDOM % 50)) bench.py --gpus 2 --steps 50 --warmup 10 --config $cfg --no-cpu-baseline --no-e2e --no-tf32 > gpurun_out/r02/combo1/nopk_$cfg.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02/combo1/nopk_$cfg.json').read().strip().splitlines()[-1]); print('nopk $cfg', round(d['ms_per_step'],4))"; done
bash scripts/r02/s3_wide.sh
