for v in k128s3w5 k64s4w8 k64s3w9 k64s6w4 k64s5w6; do
POS_LIB=/root/repo/build/libposeidon_$v.so TAG=$v timeout 120 python scripts/a4_bench.py 2>&1 | grep '^{'
done
