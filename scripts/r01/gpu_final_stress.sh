N=$(nvidia-smi -L | wc -l)
for i in 1 2 3 4; do
POS_BENCH_VERBOSE=1 POS_BENCH_WATCHDOG=80 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((33000+i)) bench.py --gpus $N --steps 50 --warmup 10 > gpurun_out/f_$i.json 2> gpurun_out/f_$i.err; rc=$?
echo "[c3 default run $i N=$N] rc=$rc $(python scripts/show_bench.py gpurun_out/f_$i.json 2>&1 | cut -c1-70)"
done
