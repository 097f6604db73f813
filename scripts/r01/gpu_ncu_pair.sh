mkdir -p gpurun_out
for v in 0 1; do
POS_SFB_PAIR=$v ncu --set full --clock-control none -k regex:sfb_tc --launch-skip 1 --launch-count 1 -o gpurun_out/pair$v -f python scripts/a4_one.py 4096,25088,32 > gpurun_out/ncu_pair$v.log 2>&1
done
ls gpurun_out
