set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python bench.py --layers > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench_rc=$?
timeout 600 python bench.py --config c1 --no-cpu-baseline --layers > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo bench_c1_rc=$?
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sfb_tc -s 3 -c 3 -o gpurun_out/prof_a4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
ls -la gpurun_out
