N=$(nvidia-smi -L | wc -l)
timeout 300 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -1
port=31600
for c in c3 c1 c2 c4; do for ss in 2 1; do
port=$((port+1))
POS_SFB_STREAMS=$ss timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] streams=$ss $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-130)"
done; done
