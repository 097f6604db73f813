# 2 GPUs: NVLink counter bytes per PS unit; NEXT-3 crossover with the Adam model column
O=gpurun_out/r02/p2bytes; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${1:-2} --master-addr 127.0.0.1"
timeout 600 $T --master-port 29931 scripts/nvlink_bytes.py $O/nvlink_bytes.json > $O/bytes.log 2>&1; echo "bytes rc=$?"; grep "^{" $O/bytes.log | cut -c1-600
timeout 600 $T --master-port 29932 scripts/scheme_crossover.py $O/scheme_crossover.json > $O/crossover.log 2>&1; echo "xover rc=$?"; tail -1 $O/crossover.log
