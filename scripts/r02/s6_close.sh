# 4 GPUs, round-2 close on the final commit: full -m gpu suite (multi-GPU tests at P = 4), smoke,
# default 1-GPU bench line, default 4-GPU bench line
O=gpurun_out/r02/close; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_4gpus.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu_4gpus.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --no-cpu-baseline > $O/bench_c3_n1.json 2> $O/bench_c3_n1.err; echo "bench n1 rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29011 bench.py --gpus 4 > $O/bench_c3_n4.json 2> $O/bench_c3_n4.err; echo "bench n4 rc=$?"
for f in $O/bench_c3_n1.json $O/bench_c3_n4.json; do python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']; print('$f', round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(r['frac'],3), round(r['step']['frac_pipelined'],3), d['e2e'] and round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
