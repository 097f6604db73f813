mkdir -p gpurun_out/final
N=$(nvidia-smi -L | wc -l)
timeout 300 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/final/pytest_multi_n$N.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/final/pytest_multi_n$N.log
grep -o '"checks".*' /tmp/x 2>/dev/null
port=31300
for c in c3 c1 c2 c4; do
port=$((port+1))
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] flags $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-60)"
port=$((port+1))
POS_GATHER_FLAGS=0 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] barrier $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-60)"
done
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 31399 bench.py --gpus $N --config c1 --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/o.json 2> gpurun_out/o.err
grep -E "SFB|PS" gpurun_out/o.err
