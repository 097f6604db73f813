N=$(nvidia-smi -L | wc -l)
port=31000
for c in 8 16 32 96; do
port=$((port+1))
POS_NVLS_CTAS=$c timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N nvls_ctas=$c $(python scripts/show_bench.py gpurun_out/o.json)"
done
port=$((port+1))
POS_NVLS_CTAS=16 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c4 --no-cpu-baseline --no-e2e --steps 30 --bucket-mb 64 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N c4 64MB nvls16 $(python scripts/show_bench.py gpurun_out/o.json)"
