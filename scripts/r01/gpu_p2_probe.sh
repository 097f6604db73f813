N=$(nvidia-smi -L | wc -l)
timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30501 scripts/sfb_unit_probe.py 2>/dev/null | grep '^{'
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30502 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --steps 30 --layers > gpurun_out/lay.json 2> gpurun_out/lay.err
python scripts/show_bench.py gpurun_out/lay.json
grep -E "PS params|SFB params" gpurun_out/lay.err | head -12
