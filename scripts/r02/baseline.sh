# round-2 baseline: isolated A4 on the bench shapes + ncu full of the CTA-pair kernel at AlexNet fc6, K*P = 1024
set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/a4_bench.py > gpurun_out/r02/a4_base.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/pair_kp1024 -f python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/ncu_pair.log 2>&1
POS_SFB_PAIR=0 ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/single_fc6 -f python scripts/a4_one.py 4096,25088,32 > gpurun_out/r02/ncu_single.log 2>&1
cat gpurun_out/r02/a4_base.txt
