mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_sched.py -q -m gpu -x > gpurun_out/pytest_multi.log 2>&1; echo pytest_rc=$?; tail -30 gpurun_out/pytest_multi.log
N=$(nvidia-smi -L | wc -l)
for c in c3 c1; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $c --no-cpu-baseline > gpurun_out/bench_${c}_n$N.json 2> gpurun_out/bench_${c}_n$N.err; echo bench_${c}_rc=$?
done
tail -5 gpurun_out/bench_c3_n$N.err
