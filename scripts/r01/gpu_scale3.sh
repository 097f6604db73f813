N=$(nvidia-smi -L | wc -l)
port=30800
for args in "" "--static-tiles" "--bucket-mb 64" "--no-symm"; do
port=$((port+1))
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 $args > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$args] $(python scripts/show_bench.py gpurun_out/o.json)"
done
for c in c1 c2 c4; do
port=$((port+1))
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] $(python scripts/show_bench.py gpurun_out/o.json)"
done
