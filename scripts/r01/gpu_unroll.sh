N=$(nvidia-smi -L | wc -l)
port=31200
for u in 4 8 16; do
POS_LIB=/root/repo/build/libposeidon_u$u.so TAG=u$u timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((port+u)) scripts/nvls_probe.py 2>/dev/null | grep '^{'
for c in c3 c4; do
port=$((port+20))
POS_LIB=/root/repo/build/libposeidon_u$u.so timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N u=$u [$c] $(python scripts/show_bench.py gpurun_out/o.json)"
done; done
