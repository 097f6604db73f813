# 2 GPUs: multi-GPU tests with the 96-CTA P = 2 PS grid, then the final P = 2 bench lines (NVLink
# peak now includes the copy-engine figure)
O=gpurun_out/r02/p2final96b; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 600 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi_p2.log 2>&1; echo "multi rc=$?"; tail -1 $O/pytest_multi_p2.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=28800
for cfg in c3 c2 c1 c4; do port=$((port+1))
  timeout 400 $T --master-port $port bench.py --gpus 2 --config $cfg > $O/bench_${cfg}_n2.json 2> $O/bench_${cfg}_n2.err
  echo "P2 $cfg rc=$? $(python -c "import json; d=json.loads(open('$O/bench_${cfg}_n2.json').read().strip().splitlines()[-1]); r=d['roofline']; print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(r['step']['frac_pipelined'],3), round(r['frac'],3), d['e2e'] and round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
done
