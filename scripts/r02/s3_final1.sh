# 1 GPU: full -m gpu suite + smoke, bench lines for every config, the reference arm, ncu launch list + A4 captures
O=gpurun_out/r02/final1; mkdir -p $O
export POS_TIMEOUT_MS=20000
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err; echo "bench c3 rc=$?"
for cfg in c1 c2 c4; do timeout 600 python bench.py --config $cfg > $O/bench_${cfg}_n1.json 2> $O/bench_${cfg}_n1.err; echo "bench $cfg rc=$?"; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_n1.json 2> $O/bench_reference_n1.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"sfb_tc|ps_apply|pack_|bias_colsum|sfb_simt" -c 60 --csv --log-file $O/launches_c3_n1.csv python bench.py --eager --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 3 --launch-count 3 -o $O/a4_c3_step -f python bench.py --eager --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o $O/a4_pair_kp1024 -f python scripts/a4_one.py 4096,9216,1024 > $O/ncu_pair.log 2>&1; echo "ncu pair rc=$?"
A4_SHAPES="4096,25088,32;21841,4096,32;4096,4096,32;4096,9216,1024;4096,4096,1024;1000,4096,1024;4096,9216,512;4096,25088,256;21841,4096,256;8192,8192,8192" timeout 300 python scripts/a4_bench.py > $O/a4_bench.txt 2>&1
POS_SFB_PAIR=1 A4_SHAPES="4096,9216,512;8192,8192,2048;8192,8192,4096;8192,8192,8192" TAG=pair_forced timeout 300 python scripts/a4_bench.py >> $O/a4_bench.txt 2>&1
cat $O/a4_bench.txt | cut -c1-200
