N=$(nvidia-smi -L | wc -l)
for c in c1 c2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] $(python scripts/show_bench.py gpurun_out/o.json)"
grep -E "^ *[0-9]+ " gpurun_out/o.err | grep -v "pack=     0.0us comm=     0.0us apply=     0.0us"
done
