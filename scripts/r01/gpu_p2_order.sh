N=$(nvidia-smi -L | wc -l)
port=30600
for args in "" "--ps-after-sfb" "--ps-after-sfb --bucket-mb 64" ""; do
port=$((port+1))
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 $args > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$args] $(python scripts/show_bench.py gpurun_out/o.json)"
done
