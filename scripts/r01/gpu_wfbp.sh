mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_torch_wfbp.py -q -m gpu -x > gpurun_out/pytest_wfbp.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/pytest_wfbp.log | grep -v "^$" | tail -25
timeout 600 python scripts/wfbp_train_bench.py --config c3 > gpurun_out/wfbp_c3.json 2> gpurun_out/wfbp_c3.err; echo rc=$?; cat gpurun_out/wfbp_c3.json; tail -5 gpurun_out/wfbp_c3.err
