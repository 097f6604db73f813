# A4 at K*P = 1024 (AlexNet fc6/fc7 at P = 8) and the VGG shapes: isolated timing with clocks, ncu full of the pair kernel
mkdir -p gpurun_out/r02/a4
(nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active,power.draw --format=csv,noheader -lms 200 > gpurun_out/r02/a4/clk.txt) & SMI=$!
A4_SHAPES="4096,9216,1024;4096,4096,1024;1000,4096,1024;4096,25088,32;21841,4096,32;4096,4096,32;4096,25088,256;21841,4096,256" timeout 300 python scripts/a4_bench.py > gpurun_out/r02/a4/pair_default.txt 2>&1
POS_SFB_PAIR=0 A4_SHAPES="4096,9216,1024;4096,9216,512" timeout 300 python scripts/a4_bench.py > gpurun_out/r02/a4/pair_off.txt 2>&1
kill $SMI
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/a4/pair_kp1024 -f python scripts/a4_one.py 4096,9216,1024 > gpurun_out/r02/a4/ncu_pair.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/r02/a4/single_fc6 -f python scripts/a4_one.py 4096,25088,32 > gpurun_out/r02/a4/ncu_single.log 2>&1
cat gpurun_out/r02/a4/pair_default.txt gpurun_out/r02/a4/pair_off.txt
sort gpurun_out/r02/a4/clk.txt | uniq -c | sort -rn | head -8
