# session-3 re-check on 1 GPU: full -m gpu suite, smoke, default bench, launch list
mkdir -p gpurun_out/r02/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/s3/smi.txt
export POS_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r02/s3/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02/s3/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/s3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02/s3/smoke.log
timeout 600 python bench.py --layers > gpurun_out/r02/s3/bench.json 2> gpurun_out/r02/s3/bench.err; echo "bench rc=$?" >> gpurun_out/r02/s3/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02/s3/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 > gpurun_out/r02/s3/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r02/s3/ncu.log
tail -3 gpurun_out/r02/s3/pytest_gpu.log gpurun_out/r02/s3/smoke.log gpurun_out/r02/s3/bench.err gpurun_out/r02/s3/ncu.log
cat gpurun_out/r02/s3/bench.json
