# A4 compile-time variants at K*P = 1024 / 512 / 32: isolated timing; parity of the new-structure variants
mkdir -p gpurun_out/r02/a4var
export A4_SHAPES="4096,9216,1024;4096,4096,1024;4096,9216,512;4096,25088,32;21841,4096,32"
for v in base exp1 exp2 pw6 pepi2pw6 ps3pw7 pepi2ps3pw8 ps2pw10 base2; do
  lib=build/libposeidon_$v.so; [ $v = base ] || [ $v = base2 ] && lib=paper_1706_03292_b200/libposeidon.so
  POS_LIB=$PWD/$lib TAG=$v timeout 200 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> gpurun_out/r02/a4var/a4.txt
done
for v in pepi2pw6 pepi2ps3pw8 ps2pw10 pw6; do
  POS_LIB=$PWD/build/libposeidon_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or kp1024 or full_size or tile_edges" > gpurun_out/r02/a4var/parity_$v.log 2>&1; echo "$v rc=$?" >> gpurun_out/r02/a4var/parity.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02/a4var/parity_base.log 2>&1; echo "base rc=$?" >> gpurun_out/r02/a4var/parity.txt
python - <<'P'
import json
for l in open("gpurun_out/r02/a4var/a4.txt"):
    d=json.loads(l); print(f"{d['tag']:12s} {d['M']:6d} {d['N']:6d} {d['KP']:5d} {d['us']:7.1f} us  frac_hbm {d['frac']:.3f}  {d['tflops']:7.1f} TF/s")
P
cat gpurun_out/r02/a4var/parity.txt
