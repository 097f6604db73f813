for c in 0 112 80 48; do
WFBP_ONLY=1 timeout 300 python scripts/wfbp_train_bench.py --config c3 --max-ctas $c 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ctas', d['max_ctas'], 'nosync %.3f wfbp %.3f exposed %.3f (%.3f)' % (d['ms_step_nosync'], d['ms_step_wfbp'], d['exposed_ms_wfbp'], d['exposed_frac_wfbp']))"
done
