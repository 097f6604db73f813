N=$(nvidia-smi -L | wc -l)
for i in 1 2 3 4 5 6; do
for c in c1 c3; do
POS_BENCH_VERBOSE=1 POS_BENCH_WATCHDOG=50 timeout 100 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((31700+i*2+${#c})) bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o_${c}_$i.json 2> gpurun_out/o_${c}_$i.err; rc=$?
echo "[$c run $i] rc=$rc $(python scripts/show_bench.py gpurun_out/o_${c}_$i.json 2>&1 | cut -c1-60)"
if [ $rc -ne 0 ]; then grep -v "^NCCL" gpurun_out/o_${c}_$i.err | grep -i "bench r\|error\|Traceback\|File \"\|Fatal\|Thread\|Timeout" | head -30; fi
done; done
