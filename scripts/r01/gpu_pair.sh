timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sched.py tests/test_gpu_guards.py -x -q 2>&1 | tail -2
for v in 0 1; do
POS_SFB_PAIR=$v TAG=pair$v timeout 120 python scripts/a4_bench.py 2>&1 | grep "^{"
done
