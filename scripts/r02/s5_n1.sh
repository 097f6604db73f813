# 1 GPU (round-2 close): full -m gpu suite, smoke, default bench line + c1/c2/c4 + f32, reference arm,
# ncu launch list of the default step
O=gpurun_out/r02/final6; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err; echo "bench rc=$?"
for c in c1 c2 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > $O/bench_${c}_n1.json 2> $O/bench_${c}_n1.err; echo "bench $c rc=$?"; done
timeout 600 python bench.py --dtype f32 --no-cpu-baseline > $O/bench_c3_n1_f32.json 2> $O/bench_c3_n1_f32.err; echo "bench f32 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_n1.json 2> $O/bench_reference_n1.err; echo "ref rc=$?"
for c in c3 c1 c2 c4 c3_n1_f32; do f=$O/bench_${c}_n1.json; [ $c = c3_n1_f32 ] && f=$O/bench_c3_n1_f32.json; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), 'frac', round(r['frac'],3), 'span', r.get('span_frac') and round(r['span_frac'],3), 'step', round(r['step']['frac_pipelined'],3), 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_c3_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 --eager > $O/ncu.log 2>&1; echo "ncu rc=$?"
