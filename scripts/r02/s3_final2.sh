# 1 GPU: full -m gpu suite, smoke, default bench line, c1 line
O=gpurun_out/r02/final2; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --config c1 --no-cpu-baseline > $O/bench_c1_n1.json 2> $O/bench_c1_n1.err; echo "bench c1 rc=$?"
for c in c3 c1; do python -c "
import json; d=json.loads(open('$O/bench_${c}_n1.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['ms_per_step'],4), d['step_stats']['median_ms'], 'frac', round(r['frac'],3), 'span_frac', round(r['span_frac'],3), r['per_layer_ms'], d['trace_timeline_us'])"; done
