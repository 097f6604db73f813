# quick check: scheduler tests + bench with the untraced timed region
mkdir -p gpurun_out/r02/check
timeout 600 python -m pytest tests/test_gpu_sched.py tests/test_gpu_parity.py -q -x > gpurun_out/r02/check/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02/check/pytest.log
for i in 1 2; do timeout 300 python bench.py --steps 50 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r02/check/bench_$i.json 2> gpurun_out/r02/check/bench_$i.err; echo "bench rc=$?"; done
tail -1 gpurun_out/r02/check/pytest.log
for i in 1 2; do python -c "import json; d=json.loads(open('gpurun_out/r02/check/bench_$i.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), round(r['kernel_ms_per_step'],4), round(r['traced_ms_per_step'],4), round(r['frac'],3), d['clocks']['sm_mhz'], d['kernels_isolated']['a2_pack'])"; done
