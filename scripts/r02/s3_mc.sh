# 4-CTA multicast A4 kernel: parity (forced on for every shape) and timing vs the pair kernel
mkdir -p gpurun_out/r02/mc
export POS_TIMEOUT_MS=20000
POS_SFB_PAIR=1 POS_SFB_MC=1 POS_SFB_VERBOSE=1 timeout 300 python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/mc/one.log 2>&1; echo "one rc=$?" >> gpurun_out/r02/mc/one.log
cat gpurun_out/r02/mc/one.log
if grep -q "one rc=0" gpurun_out/r02/mc/one.log; then
POS_SFB_PAIR=1 POS_SFB_MC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair or kp1024 or full_size or tile_edges or c0_sfb" > gpurun_out/r02/mc/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/r02/mc/parity.log
tail -3 gpurun_out/r02/mc/parity.log
export A4_SHAPES="4096,9216,1024;4096,4096,1024;1000,4096,1024;4096,9216,512;4096,25088,256;21841,4096,256;4096,9216,2048"
for mc in 1 0 1 0; do POS_SFB_PAIR=1 POS_SFB_MC=$mc TAG=mc$mc timeout 300 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> gpurun_out/r02/mc/a4.txt; done
python - <<'P'
import json
for l in open("gpurun_out/r02/mc/a4.txt"):
    d=json.loads(l); print(f"{d['tag']:6s} {d['M']:6d} {d['N']:6d} {d['KP']:5d} {d['us']:7.1f} us  frac_hbm {d['frac']:.3f}  {d['tflops']:7.1f} TF/s")
P
POS_SFB_PAIR=1 POS_SFB_MC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/mc/mc_kp1024 -f python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/mc/ncu.log 2>&1
fi
