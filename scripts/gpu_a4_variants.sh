for v in n256s3w5 n128s3w8 n128s2w10; do
POS_LIB=/root/repo/build/libposeidon_$v.so TAG=$v timeout 120 python scripts/a4_bench.py 2>&1 | grep '^{'
done
