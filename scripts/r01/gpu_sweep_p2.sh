mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
port=29600
for ctas in 16 32; do for mb in 2 16 64; do
port=$((port+1))
POS_NCCL_MAX_CTAS=$ctas timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --bucket-mb $mb --steps 30 > gpurun_out/sw_${ctas}_${mb}.json 2> gpurun_out/sw_${ctas}_${mb}.err
echo "ctas=$ctas mb=$mb rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sw_${ctas}_${mb}.json'));print(round(d['ms_per_step'],4), round(d['eager_ms_per_step'],4), d['config']['ps_units'])" 2>&1)"
done; done
