mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sched.py -q -m gpu -x > gpurun_out/pytest_gpu_sched.log 2>&1; echo pytest_rc=$?; tail -15 gpurun_out/pytest_gpu_sched.log
for c in c3 c1 c2 c4; do
timeout 600 python bench.py --config $c --layers --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?
done
tail -5 gpurun_out/bench_c3.err
