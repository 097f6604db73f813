N=$(nvidia-smi -L | wc -l)
TAG=default timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30901 scripts/nvls_probe.py 2>/dev/null | grep '^{'
POS_NCCL_MAX_CTAS=32 TAG=nccl32 timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30902 scripts/nvls_probe.py 2>/dev/null | grep '^{'
