mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
port=29900
for ctas in 128 148; do for mb in 16 32; do
port=$((port+1))
POS_SFB_MAX_CTAS=$ctas timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --bucket-mb $mb > gpurun_out/sw.json 2> gpurun_out/sw.err
echo "ctas=$ctas mb=$mb rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sw.json'));print(round(d['ms_per_step'],4), round(d['eager_ms_per_step'],4), d['config']['ps_units'])" 2>&1 | tail -1)"
done; done
POS_SFB_MAX_CTAS=148 timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29950 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --bucket-mb 16 --layers > gpurun_out/lay.json 2> gpurun_out/lay.err
grep -E "PS params|SFB params" gpurun_out/lay.err | head -12
