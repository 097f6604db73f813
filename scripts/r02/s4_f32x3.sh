# 2 GPUs: full GPU suite (incl. the P = 2 multi tests: f32 barrier-mode gather, now 3xTF32 rows),
# then 1-GPU bench lines for f32 (3xTF32 tensor-core reconstruction) and the default bf16 step
O=gpurun_out/r02/f32x3; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -q -m gpu -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
for d in f32 bf16; do
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --dtype $d --no-cpu-baseline > $O/bench_$d.json 2> $O/bench_$d.err; echo "$d rc=$?"
  python -c "import json; d=json.loads(open('$O/bench_$d.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), r['frac'], r['kernels_isolated']['a4_reconstruct_apply'])"
done
