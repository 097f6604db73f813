N=$(nvidia-smi -L | wc -l)
timeout 400 python -m pytest tests/test_gpu_multi.py -q -m gpu -x 2>&1 | tail -1
for v in 0 1; do
POS_PS_P2P=$v PROBE_MB=0.0625,4,19,80 TAG=p2p$v timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29570+v)) scripts/nvls_probe.py 2>/dev/null | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'].ljust(6), str(d['MB']).rjust(7), 'MB ps', str(d['nvls_us']).rjust(7), 'us  allreduce', d['torch_allreduce_us'])"
done
port=32300
for c in c4 c2 c3; do for v in 1 0; do
port=$((port+1))
POS_PS_P2P=$v timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] p2p=$v $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-50)"
done; done
