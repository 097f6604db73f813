# 4-GPU box (round-2 close, after 3xTF32 / epoch barriers / auto pack placement): final multi-GPU tests at P=4 and P=2, full default bench lines at P=2 and P=4
O=gpurun_out/r02/final5; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi_p4.log 2>&1; echo "multi p4 rc=$?" >> $O/pytest_multi_p4.log; tail -2 $O/pytest_multi_p4.log
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi_p2.log 2>&1; echo "multi p2 rc=$?" >> $O/pytest_multi_p2.log; tail -2 $O/pytest_multi_p2.log
port=29990
for N in 4 2; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  for cfg in c3 c1 c2 c4; do port=$((port+1))
    timeout 400 $T --master-port $port bench.py --gpus $N --config $cfg > $O/bench_${cfg}_n$N.json 2> $O/bench_${cfg}_n$N.err
    echo "P$N $cfg rc=$? $(python -c "import json; d=json.loads(open('$O/bench_${cfg}_n$N.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(r['step']['frac_pipelined'],3), round(r['frac'],3), d['e2e'] and round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
