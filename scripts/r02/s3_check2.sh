# 1 GPU after the A4 cleanup: parity suites, A4 timing at K*P = 32 / 1024, default bench
O=gpurun_out/r02/check2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py tests/test_gpu_loopback.py tests/test_gpu_guards.py -q -x > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
A4_SHAPES="4096,25088,32;21841,4096,32;4096,9216,1024;4096,4096,1024" timeout 300 python scripts/a4_bench.py 2>&1 | grep '^{' | grep -v '"M": [01],' | cut -c1-160
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-tf32 > $O/bench.json 2>/dev/null; python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
