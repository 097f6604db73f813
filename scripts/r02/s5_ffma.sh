# 1 GPU: exact-fp32 mode (POS_F32_FFMA=1) vs the 3xTF32 default on every f32 GPU test, and an f32 bench line in each mode
O=gpurun_out/r02/ffma; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_guards.py tests/test_gpu_sched.py -q -k f32 > $O/pytest_f32_3xtf32.log 2>&1; echo "3xtf32 rc=$?"; tail -1 $O/pytest_f32_3xtf32.log
POS_F32_FFMA=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_guards.py tests/test_gpu_sched.py -q -k f32 > $O/pytest_f32_ffma.log 2>&1; echo "ffma rc=$?"; tail -1 $O/pytest_f32_ffma.log
POS_F32_FFMA=1 timeout 600 python bench.py --dtype f32 --no-cpu-baseline --no-e2e > $O/bench_f32_ffma.json 2> $O/bench_f32_ffma.err; echo "bench ffma rc=$?"
python -c "import json; d=json.loads(open('$O/bench_f32_ffma.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), d['roofline']['kernels_isolated']['a4_reconstruct_apply']['us'])"
