mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
echo "GPUs: $N"
nvidia-smi topo -m | head -3
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/pytest_multi_n$N.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_multi_n$N.log
port=30100
for args in "--bucket-mb 2" "--bucket-mb 16" "--bucket-mb 64" "--no-symm --bucket-mb 16"; do
port=$((port+1))
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 $args > gpurun_out/sc.json 2> gpurun_out/sc.err
echo "N=$N $args rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sc.json'));r=d['roofline'];print(round(d['ms_per_step'],4), round(d['eager_ms_per_step'],4), d['config']['ps_units'], 'roof', round(r['step']['t_roofline_pipelined_ms'],4), 'a4', round(r['achieved']), 'val %.3g'%d['value'])" 2>&1 | tail -1)"
done
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30190 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --bucket-mb 16 --layers > gpurun_out/sc_layers.json 2> gpurun_out/sc_layers.err
grep -E "PS params|SFB params" gpurun_out/sc_layers.err | head -12
for c in c1 c2 c4; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 3020${c: -1} bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 30 --bucket-mb 16 > gpurun_out/sc_$c.json 2> gpurun_out/sc_$c.err
echo "N=$N $c rc=$? $(python -c "import json;d=json.load(open('gpurun_out/sc_$c.json'));r=d['roofline'];print(round(d['ms_per_step'],4), round(d['eager_ms_per_step'],4), 'roof', round(r['step']['t_roofline_pipelined_ms'],4), 'val %.3g'%d['value'])" 2>&1 | tail -1)"
done
