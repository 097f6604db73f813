N=$(nvidia-smi -L | wc -l)
NCCL_DEBUG=INFO timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 scripts/nvls_probe.py > gpurun_out/nv.out 2> gpurun_out/nv.err
grep '^{' gpurun_out/nv.out
grep -i "nvls" gpurun_out/nv.err | head -5
grep -i "algo\|protocol\|Channel" gpurun_out/nv.err | head -5
