# 2 GPUs: loopback re-check, multi-GPU tests, NVLink peaks at P=2, bench N=1 and N=2
mkdir -p gpurun_out/r02
export POS_TIMEOUT_MS=20000
timeout 300 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/r02/pytest_loop.log 2>&1; echo "loop rc=$?" >> gpurun_out/r02/pytest_loop.log
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q -s > gpurun_out/r02/pytest_multi_n2.log 2>&1; echo "multi rc=$?" >> gpurun_out/r02/pytest_multi_n2.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/nvlink_peaks.py > gpurun_out/r02/nvlink_p2.log 2>&1; echo "nvl rc=$?" >> gpurun_out/r02/nvlink_p2.log
cp profiles/nvlink_peaks.json gpurun_out/r02/nvlink_peaks.json 2>/dev/null
timeout 600 python bench.py --steps 30 --warmup 5 --layers > gpurun_out/r02/bench_c3_n1.json 2> gpurun_out/r02/bench_c3_n1.err; echo "b1 rc=$?" >> gpurun_out/r02/bench_c3_n1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 30 --warmup 5 --layers > gpurun_out/r02/bench_c3_n2.json 2> gpurun_out/r02/bench_c3_n2.err; echo "b2 rc=$?" >> gpurun_out/r02/bench_c3_n2.err
tail -2 gpurun_out/r02/pytest_loop.log gpurun_out/r02/pytest_multi_n2.log gpurun_out/r02/nvlink_p2.log gpurun_out/r02/bench_c3_n1.err gpurun_out/r02/bench_c3_n2.err
