N=$(nvidia-smi -L | wc -l)
for nv in $NVS; do for c in c3 c2; do
POS_NVLS_CTAS=$nv timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((32800+nv+${c:1:1})) bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] nvls_ctas=$nv $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
done; done
