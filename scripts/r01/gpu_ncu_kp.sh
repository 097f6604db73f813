mkdir -p gpurun_out
python scripts/a4_one.py 4096,25088,256 4096,9216,1024 || exit 1
ncu --set full --clock-control none -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/kp256 -f python scripts/a4_one.py 4096,25088,256 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/kp1024 -f python scripts/a4_one.py 4096,9216,1024 > gpurun_out/ncu2.log 2>&1
ls -la gpurun_out
