mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for c in c3 c1 c2 c4; do
timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_${c}_rc=$?
done
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --layers > gpurun_out/bench_c3_layers.json 2> gpurun_out/bench_c3_layers.err
grep -E "PS params|SFB params" gpurun_out/bench_c3_layers.err
