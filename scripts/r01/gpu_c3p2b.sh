N=$(nvidia-smi -L | wc -l)
for nv in 32 16 64 8; do
POS_NVLS_CTAS=$nv timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((32710+nv)) bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [c3] nvls_ctas=$nv $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
done
