POS_SFB_PAIR=1 POS_BENCH_VERBOSE=1 POS_BENCH_WATCHDOG=60 timeout 120 python bench.py --config c1 --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/o.json 2> gpurun_out/o.err; echo rc=$?
tail -20 gpurun_out/o.err
python scripts/show_bench.py gpurun_out/o.json | cut -c1-100
