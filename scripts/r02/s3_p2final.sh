# 2 GPUs, final defaults: multi-GPU tests, NVLink peaks (incl. the P=2 peer kernel), full bench lines
O=gpurun_out/r02/p2final; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q -s > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log; tail -2 $O/pytest_multi.log
timeout 400 $T --master-port 29511 scripts/nvlink_peaks.py $O/nvlink_peaks.json > $O/nvlink.log 2>&1; echo "nvl rc=$?"
port=29880
for cfg in c3 c1 c2 c4; do port=$((port+1)); timeout 400 $T --master-port $port bench.py --gpus 2 --config $cfg > $O/bench_${cfg}_n2.json 2> $O/bench_${cfg}_n2.err; echo "$cfg rc=$? $(python -c "import json; d=json.loads(open('$O/bench_${cfg}_n2.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(d['roofline']['step']['frac_pipelined'],3), d['e2e'] and round(d['e2e']['ms_per_step'],3))")"; done
