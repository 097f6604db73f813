N=$(nvidia-smi -L | wc -l)
port=29960
for v in eacq_rel erelaxed default; do
L=/root/repo/build/libposeidon_$v.so; [ $v = default ] && L=/root/repo/paper_1706_03292_b200/libposeidon.so
port=$((port+1))
POS_LIB=$L PROBE_MB=0.0625,4,19 TAG=$v timeout 200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port scripts/nvls_probe.py 2>/dev/null | grep '^{' | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); print(d['tag'].ljust(9), str(d['MB']).rjust(7), 'MB nvls', str(d['nvls_us']).rjust(7))"
for c in c3 c4 c1; do
port=$((port+1))
POS_LIB=$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
echo "N=$N [$c] $v $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-50)"
done; done
