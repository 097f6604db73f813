mkdir -p gpurun_out/final
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/final/pytest_multi_n$N.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/final/pytest_multi_n$N.log
port=31100
for c in c3 c1 c2 c4; do
port=$((port+1))
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c --no-cpu-baseline > gpurun_out/final/scale_${c}_n$N.json 2> gpurun_out/final/scale_${c}_n$N.err
echo "N=$N [$c] $(python scripts/show_bench.py gpurun_out/final/scale_${c}_n$N.json)"
done
