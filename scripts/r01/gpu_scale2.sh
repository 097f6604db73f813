mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
port=30300
for env in "POS_NVLS_CTAS=32" "POS_NVLS_CTAS=96" "POS_NVLS_CTAS=128" "POS_NVLS_CTAS=96 POS_SFB_MAX_CTAS=128"; do for mb in 16; do
port=$((port+1))
env $env timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --bucket-mb $mb > gpurun_out/sc.json 2> gpurun_out/sc.err
echo "N=$N $env mb=$mb rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sc.json'));r=d['roofline'];print(round(d['ms_per_step'],4), round(d['eager_ms_per_step'],4), d['config']['ps_units'], 'a4', round(r['achieved']), 'ps', round(r['ps_apply']['achieved_gbs']))" 2>&1 | tail -1)"
done; done
POS_NVLS_CTAS=96 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30390 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --bucket-mb 16 --layers > gpurun_out/sc_layers.json 2> gpurun_out/sc_layers.err
grep -E "PS params|SFB params" gpurun_out/sc_layers.err | head -12
