mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/pytest_multi.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/pytest_multi.log | grep -v "^$" | tail -25
