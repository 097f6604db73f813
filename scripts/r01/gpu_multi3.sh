mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
export POS_BENCH_VERBOSE=1 POS_BENCH_WATCHDOG=100
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config c3 --no-cpu-baseline > gpurun_out/bench_c3_n$N.json 2> gpurun_out/bench_c3_n$N.err; echo graph_rc=$?
grep "bench r\|Thread\|File" gpurun_out/bench_c3_n$N.err | head -30
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --config c3 --no-cpu-baseline --no-e2e --eager --layers --steps 20 > gpurun_out/dbg_eager.json 2> gpurun_out/dbg_eager.err; echo eager_rc=$?
grep -v "^W1018\|elastic\|\*\*\*\|OMP\|bench r" gpurun_out/dbg_eager.err | tail -20
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --config c1 --no-cpu-baseline > gpurun_out/bench_c1_n$N.json 2> gpurun_out/bench_c1_n$N.err; echo c1_rc=$?
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus $N --config c4 --no-cpu-baseline > gpurun_out/bench_c4_n$N.json 2> gpurun_out/bench_c4_n$N.err; echo c4_rc=$?
