# A4 diagnostics at K*P = 1024: no-operand variant timing, ncu of the no-MMA variant; bench with the untraced timed region
mkdir -p gpurun_out/r02/a4diag
export A4_SHAPES="4096,9216,1024;4096,9216,512;4096,25088,32"
for v in exp3 exp2; do POS_LIB=$PWD/build/libposeidon_$v.so TAG=$v timeout 200 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> gpurun_out/r02/a4diag/a4.txt; done
POS_LIB=$PWD/build/libposeidon_exp2.so timeout 600 ncu --set full --clock-control none -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/a4diag/exp2_kp1024 -f python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/a4diag/ncu_exp2.log 2>&1
POS_LIB=$PWD/build/libposeidon_exp3.so timeout 600 ncu --set full --clock-control none -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/a4diag/exp3_kp1024 -f python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/a4diag/ncu_exp3.log 2>&1
timeout 600 python -m pytest tests/test_gpu_sched.py -q -x > gpurun_out/r02/a4diag/pytest_sched.log 2>&1; echo "sched rc=$?" >> gpurun_out/r02/a4diag/pytest_sched.log
for i in 1 2; do timeout 300 python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02/a4diag/bench_$i.json 2> gpurun_out/r02/a4diag/bench_$i.err; echo "bench rc=$?"; done
cat gpurun_out/r02/a4diag/a4.txt; tail -1 gpurun_out/r02/a4diag/pytest_sched.log
for i in 1 2; do python -c "import json; d=json.loads(open('gpurun_out/r02/a4diag/bench_$i.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), round(r['kernel_ms_per_step'],4), round(r['traced_ms_per_step'],4), round(r['frac'],3), d['clocks']['sm_mhz'])"; done
