mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/pytest_multi.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_multi.log
port=29800
for args in "--bucket-mb 2" "--bucket-mb 16" "--bucket-mb 64" "--no-symm --bucket-mb 64"; do
port=$((port+1))
POS_NCCL_MAX_CTAS=32 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 $args > gpurun_out/sw.json 2> gpurun_out/sw.err
echo "$args rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],4), round(d['eager_ms_per_step'],4), d['config']['ps_units'], d['config']['collectives'])" 2>&1 | tail -1)"
done
