N=$(nvidia-smi -L | wc -l)
for c in 32 96 128; do
POS_NVLS_CTAS=$c TAG=ctas$c timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 3070${c: -1} scripts/nvls_probe.py 2>/dev/null | grep '^{'
done
