# wide CTA-pair A4 tile (256 x 512): parity forced on every shape; timing vs the 256 x 256 pair kernel
mkdir -p gpurun_out/r02/wide
POS_SFB_PAIR=1 POS_SFB_WIDE=1 POS_SFB_VERBOSE=1 timeout 120 python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/wide/one.log 2>&1; echo "one rc=$?" >> gpurun_out/r02/wide/one.log
cat gpurun_out/r02/wide/one.log
if grep -q "one rc=0" gpurun_out/r02/wide/one.log; then
POS_SFB_PAIR=1 POS_SFB_WIDE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or kp1024 or full_size or tile_edges or c0_sfb" > gpurun_out/r02/wide/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/r02/wide/parity.log
tail -3 gpurun_out/r02/wide/parity.log
export A4_SHAPES="4096,9216,1024;4096,4096,1024;1000,4096,1024;4096,9216,512;4096,9216,2048;4096,25088,256"
for v in base w35 w34; do
  lib=build/libposeidon_$v.so; [ $v = base ] && lib=paper_1706_03292_b200/libposeidon.so
  for wd in 1 0; do POS_LIB=$PWD/$lib POS_SFB_PAIR=1 POS_SFB_WIDE=$wd TAG=${v}_w$wd timeout 300 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> gpurun_out/r02/wide/a4.txt; done
done
python - <<'P'
import json
for l in open("gpurun_out/r02/wide/a4.txt"):
    d=json.loads(l); print(f"{d['tag']:8s} {d['M']:6d} {d['N']:6d} {d['KP']:5d} {d['us']:7.1f} us  frac_hbm {d['frac']:.3f}  {d['tflops']:7.1f} TF/s")
P
fi
