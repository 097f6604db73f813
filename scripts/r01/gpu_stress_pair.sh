N=$(nvidia-smi -L | wc -l)
for i in 1 2 3 4 5 6 7 8; do
POS_SFB_PAIR_KP=512 POS_BENCH_VERBOSE=1 POS_BENCH_WATCHDOG=50 timeout 100 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((32600+i)) bench.py --gpus $N --config c1 --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/p_$i.json 2> gpurun_out/p_$i.err; rc=$?
echo "[c1 pair single-stream run $i N=$N] rc=$rc $(python scripts/show_bench.py gpurun_out/p_$i.json 2>&1 | cut -c1-60)"
done
