mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
for args in "" "--static-tiles"; do for c in c3 c1; do
timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e $args > gpurun_out/d.json 2> gpurun_out/d.err; echo "[$c $args] $(python scripts/show_bench.py gpurun_out/d.json)"
done; done
