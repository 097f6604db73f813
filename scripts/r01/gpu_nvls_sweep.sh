N=$(nvidia-smi -L | wc -l)
port=29900
for u in 4 8; do for c in 16 32 64 128; do
port=$((port+1))
POS_LIB=/root/repo/build/libposeidon_u$u.so POS_NVLS_CTAS=$c TAG=u${u}c$c timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port scripts/nvls_probe.py 2>/dev/null | grep '^{'
done; done
