timeout 600 python -m pytest tests/test_gpu_sched.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for c in c1 c2 c3 c4; do
timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/o.json 2> gpurun_out/o.err
echo "[$c] $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-150)"
python -c "import json; d=json.load(open('gpurun_out/o.json')); print('   ', d['roofline']['kernel_ms_per_step'], d['roofline']['kernel_ms_note'], d['gpu_launches'])"
done
