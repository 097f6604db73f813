mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,GRAPH,TUNING timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29521 scripts/nccl_probe.py > gpurun_out/nccl_probe.txt 2> gpurun_out/nccl_probe.err; echo rc=$?
grep "^{" gpurun_out/nccl_probe.txt
grep -iE "via P2P|NVLS|P2P/|Channel 00|nvls|transport|CUMEM|Using network|comm 0x.*rank 0 nRanks" gpurun_out/nccl_probe.txt gpurun_out/nccl_probe.err | head -30
