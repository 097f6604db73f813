for m in 8 4 2; do for c in c4 c3; do
POS_STREAM_CTAS_PER_SM=$m timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/o.json 2> gpurun_out/o.err
echo "[$c] cap=${m}x $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-60)"
done; done
