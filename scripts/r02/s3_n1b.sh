# 1 GPU: compute-sanitizer on the small-shape script; P=1 bench with 64 vs 16 MiB buckets
O=gpurun_out/r02/n1b; mkdir -p $O
timeout 120 python scripts/sanitize_small.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -1 $O/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py > $O/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 $O/san_$tool.log
done
for cfg in c3 c1 c2 c4; do
  for b in 64 16; do timeout 300 python bench.py --config $cfg --bucket-mb $b --no-cpu-baseline --no-e2e --no-tf32 > $O/b${b}_$cfg.json 2>/dev/null; echo "$cfg b$b $(python -c "import json; d=json.loads(open('$O/b${b}_$cfg.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))")"; done
done
