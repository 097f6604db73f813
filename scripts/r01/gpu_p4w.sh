N=$(nvidia-smi -L | wc -l)
port=32400
for c in c3 c2; do for v in default s2w7 s2w6 s3w4; do
L=/root/repo/build/libposeidon_$v.so; [ $v = default ] && L=/root/repo/paper_1706_03292_b200/libposeidon.so
port=$((port+1))
POS_LIB=$L timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] $v $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-50)"
done; done
