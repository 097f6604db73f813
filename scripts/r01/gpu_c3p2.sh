N=$(nvidia-smi -L | wc -l)
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 32700 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [c3] layers: $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
grep -E "SFB|PS" gpurun_out/o.err | sed 's/  */ /g' | cut -c1-100
for v in 1 0; do
POS_GATHER_FLAGS=$v timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((32701+v)) bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [c3] flags=$v $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
done
POS_SFB_STREAMS=1 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 32705 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [c3] 1 stream $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-40)"
