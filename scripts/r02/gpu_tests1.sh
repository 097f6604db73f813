# 1-GPU: the whole -m gpu suite (driver's GPUTEST configuration), new tests first
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/smi.txt
timeout 600 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_sched.py tests/test_gpu_torch_wfbp.py -x -q > gpurun_out/r02/pytest_new.log 2>&1
echo "new rc=$?" >> gpurun_out/r02/pytest_new.log
timeout 900 python -m pytest tests/test_gpu_fullmodel.py -x -q --durations=10 > gpurun_out/r02/pytest_full.log 2>&1
echo "full rc=$?" >> gpurun_out/r02/pytest_full.log
timeout 1200 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02/pytest_gpu_n1.log 2>&1
echo "all rc=$?" >> gpurun_out/r02/pytest_gpu_n1.log
tail -3 gpurun_out/r02/pytest_new.log gpurun_out/r02/pytest_full.log gpurun_out/r02/pytest_gpu_n1.log
