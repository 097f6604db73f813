# 1 GPU: loopback tests incl. P = 3 / 16, exact-fp32 (SIMT) bench line
O=gpurun_out/r02/misc; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_loopback.py -q > $O/pytest_loop.log 2>&1; echo "loop rc=$?"; tail -1 $O/pytest_loop.log
timeout 600 python bench.py --dtype f32 --no-cpu-baseline --no-e2e > $O/bench_f32.json 2> $O/bench_f32.err; echo "f32 rc=$?"
python -c "import json; d=json.loads(open('$O/bench_f32.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), r['per_layer_ms'], r['kernels_isolated']['a4_reconstruct_apply'])"
