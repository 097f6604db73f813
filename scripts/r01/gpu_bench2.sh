mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --layers --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_rc=$?
timeout 600 python bench.py --layers --no-cpu-baseline --no-e2e --sequential > gpurun_out/bench_c3_seq.json 2> gpurun_out/bench_c3_seq.err; echo bench_rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline --layers --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1_rc=$?
timeout 600 python bench.py --config c4 --no-cpu-baseline --layers --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_c4_rc=$?
