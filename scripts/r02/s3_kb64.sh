# 64-byte K stages (finer operand ring) for both kernels vs the default
O=gpurun_out/r02/kb64; mkdir -p $O
export A4_SHAPES="4096,25088,32;21841,4096,32;4096,9216,512;4096,9216,1024;4096,4096,1024;4096,9216,2048"
for v in base kb64 kb64p9 base2; do
  lib=build/libposeidon_$v.so; case $v in base*) lib=paper_1706_03292_b200/libposeidon.so;; esac
  POS_LIB=$PWD/$lib TAG=$v timeout 200 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> $O/a4.txt
done
python - <<'P'
import json
for l in open("gpurun_out/r02/kb64/a4.txt"):
    d=json.loads(l); print(f"{d['tag']:8s} {d['M']:6d} {d['N']:6d} {d['KP']:5d} {d['us']:7.1f} us  frac_hbm {d['frac']:.3f}  {d['tflops']:7.1f} TF/s")
P
