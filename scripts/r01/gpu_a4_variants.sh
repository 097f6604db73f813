export POS_SFB_PAIR=1
export A4_SHAPES="4096,25088,32;4096,25088,256;4096,9216,512;4096,9216,1024;4096,4096,1024"
for v in p4w5 p5w4 p6w2; do
POS_LIB=/root/repo/build/libposeidon_$v.so TAG=$v timeout 120 python scripts/a4_bench.py 2>&1 | grep "^{"
done
