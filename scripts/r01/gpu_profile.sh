mkdir -p gpurun_out/prof
for c in c3 c1 c2 c4; do
timeout 300 python bench.py --config $c > gpurun_out/prof/bench_$c.json 2> gpurun_out/prof/bench_$c.err; echo bench_${c}_rc=$?
done
# launch list: skip setup (weights init etc.), capture a window of the timed region (eager so kernels are visible)
timeout 300 python bench.py --config c3 --eager --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"pos::" -s 60 -c 120 --csv --log-file gpurun_out/prof/launches_c3.csv python bench.py --config c3 --eager --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu1.log 2>&1; echo ncu1=$?
timeout 300 python bench.py --config c3 --eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sfb_tc|ps_apply_vec|pack_bf16" -s 20 -c 6 -o gpurun_out/prof/full_c3 python bench.py --config c3 --eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu2.log 2>&1; echo ncu2=$?
