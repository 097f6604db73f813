mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sched.py -q -m gpu -x > gpurun_out/pytest_gpu_sched.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu_sched.log
for c in c3 c1 c2 c4; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?
done
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --bucket-mb 0 > gpurun_out/bench_c3_nobucket.json 2> gpurun_out/bench_c3_nobucket.err; echo rc=$?
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --layers > gpurun_out/bench_c3_layers.json 2> gpurun_out/bench_c3_layers.err; echo rc=$?
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e --layers > gpurun_out/bench_c4_layers.json 2> gpurun_out/bench_c4_layers.err; echo rc=$?
tail -3 gpurun_out/bench_c3.err
