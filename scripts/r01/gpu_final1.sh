# Round-end measurement set on ONE GPU: tests, smoke, bench (all configs), reference arm,
# ncu launch list of the timed region and one --set full capture of the A4 launches.
mkdir -p gpurun_out/final
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/final/smoke.log
timeout 400 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo bench_default_rc=$?
for c in c1 c2 c4; do
timeout 300 python bench.py --config $c > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err; echo bench_${c}_rc=$?
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo ref_rc=$?
python scripts/show_bench.py gpurun_out/final/bench_default.json gpurun_out/final/bench_c1.json gpurun_out/final/bench_c2.json gpurun_out/final/bench_c4.json
timeout 300 python bench.py --config c3 --eager --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sfb_tc|ps_apply|pack_|bias_colsum|sfb_simt" -s 30 -c 50 --csv --log-file gpurun_out/final/launches_c3.csv python bench.py --config c3 --eager --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu1.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sfb_tc" -s 9 -c 3 -o gpurun_out/final/full_c3_a4 -f python bench.py --config c3 --eager --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/ncu2.log 2>&1; echo ncu2=$?
ls -la gpurun_out/final
