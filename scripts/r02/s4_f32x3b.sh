# 2 GPUs: full GPU suite after the 3xTF32 change (guard test slot sizes fixed)
O=gpurun_out/r02/f32x3; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" $O/pytest_gpu2.log | tail -8
