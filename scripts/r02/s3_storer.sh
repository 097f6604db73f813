# storer-thread variants of A4 vs base, single and pair kernels; parity of the storer build
O=gpurun_out/r02/storer; mkdir -p $O
export A4_SHAPES="4096,25088,32;21841,4096,32;4096,4096,32;4096,9216,512;4096,25088,256;4096,9216,1024;4096,4096,1024;4096,9216,2048"
for v in base st stw4 ps5pw4 stps5pw4 stps5pw3 base2; do
  lib=build/libposeidon_$v.so; case $v in base*) lib=paper_1706_03292_b200/libposeidon.so;; esac
  POS_LIB=$PWD/$lib TAG=$v timeout 200 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> $O/a4.txt
done
python - <<'P'
import json
for l in open("gpurun_out/r02/storer/a4.txt"):
    d=json.loads(l); print(f"{d['tag']:9s} {d['M']:6d} {d['N']:6d} {d['KP']:5d} {d['us']:7.1f} us  frac_hbm {d['frac']:.3f}  {d['tflops']:7.1f} TF/s")
P
for v in stps5pw4; do
  POS_LIB=$PWD/build/libposeidon_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $O/parity_$v.log 2>&1; echo "$v rc=$?" >> $O/parity.txt
  POS_LIB=$PWD/build/libposeidon_$v.so POS_SFB_PAIR=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or kp1024 or full_size or tile_edges or c0_sfb" > $O/parity_pair_$v.log 2>&1; echo "$v pair rc=$?" >> $O/parity.txt
done
cat $O/parity.txt
