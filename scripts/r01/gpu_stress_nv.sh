N=$(nvidia-smi -L | wc -l)
for i in 1 2 3 4 5 6 7 8; do
c=c3; [ $((i % 4)) -eq 0 ] && c=c2
POS_NVLS_CTAS=64 POS_BENCH_VERBOSE=1 POS_BENCH_WATCHDOG=50 timeout 100 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((32900+i)) bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/n_$i.json 2> gpurun_out/n_$i.err; rc=$?
echo "[$c nv64 run $i N=$N] rc=$rc $(python scripts/show_bench.py gpurun_out/n_$i.json 2>&1 | cut -c1-50)"
[ $rc -ne 0 ] && grep -v "^NCCL" gpurun_out/n_$i.err | grep -i "error\|Timeout\|line [0-9]* in" | head -8
done
