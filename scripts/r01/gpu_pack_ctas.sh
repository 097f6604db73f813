N=$(nvidia-smi -L | wc -l)
port=29950
for c in c1 c3; do for lib in paper_1706_03292_b200/libposeidon.so build/libposeidon_w4.so; do
port=$((port+1))
POS_LIB=/root/repo/$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] $lib $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-60)"
grep -E "SFB|PS" gpurun_out/o.err | awk '{print "    ", $2, $5, $6, $7, $8, $9}'
done; done
