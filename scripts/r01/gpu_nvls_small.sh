N=$(nvidia-smi -L | wc -l)
PROBE_MB=0.0625,0.25,1,4 TAG=c32 timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 scripts/nvls_probe.py 2>/dev/null | grep '^{'
POS_NVLS_CTAS=1 PROBE_MB=0.0625,0.25,1,4 TAG=c1 timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29556 scripts/nvls_probe.py 2>/dev/null | grep '^{'
