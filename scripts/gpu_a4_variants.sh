for v in h0 h1; do
POS_LIB=/root/repo/build/libposeidon_$v.so TAG=$v timeout 120 python scripts/a4_bench.py 2>&1 | grep '^{'
done
for v in h0 h1; do
POS_LIB=/root/repo/build/libposeidon_$v.so timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e > gpurun_out/d.json 2>/dev/null; echo "[$v] $(python scripts/show_bench.py gpurun_out/d.json)"
done
