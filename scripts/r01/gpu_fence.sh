N=$(nvidia-smi -L | wc -l)
port=32100
for c in c1 c3; do for pc in 128 296 592; do
port=$((port+1))
POS_PACK_CTAS_FLAG=$pc timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] pc=$pc layers: $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
grep -E "SFB" gpurun_out/o.err | sed 's/  */ /g' | cut -c1-90
port=$((port+1))
POS_PACK_CTAS_FLAG=$pc timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] pc=$pc $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
done; done
