N=$(nvidia-smi -L | wc -l)
port=31500
for c in c1 c3; do for uc in 0 1; do
port=$((port+1))
POS_PACK_UC=$uc timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] uc=$uc layers: $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
grep -E "SFB" gpurun_out/o.err | awk '{print "    ", $2, $5, $6}'
port=$((port+1))
POS_PACK_UC=$uc timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] uc=$uc $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
done; done
