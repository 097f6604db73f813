# 2 GPUs: one PS unit alone, copy engines vs the fused kernel
O=gpurun_out/r02/ce; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${1:-2} --master-addr 127.0.0.1"
for ce in 1 0; do timeout 300 env POS_PS_CE=$ce $T --master-port 2977$ce scripts/ps_unit_bench.py 1 4 16 64 256 2>&1 | grep -v Warn | tail -6; done
