# N GPUs (N = $1, default 2): multi-GPU tests, NVLink peaks, bench lines for every config, stress with the P=8 settings
N=${1:-2}
O=gpurun_out/r02/p$N
mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q -s > $O/pytest_multi.log 2>&1; echo "multi rc=$?" >> $O/pytest_multi.log
timeout 400 $T --master-port 29511 scripts/nvlink_peaks.py $O/nvlink_peaks.json > $O/nvlink.log 2>&1; echo "nvl rc=$?" >> $O/nvlink.log
port=29520
for cfg in c3 c1 c2 c4; do
  port=$((port+1))
  timeout 400 $T --master-port $port bench.py --gpus $N --steps 50 --warmup 10 --config $cfg --layers --no-cpu-baseline > $O/bench_$cfg.json 2> $O/bench_$cfg.err; echo "bench $cfg rc=$?" >> $O/bench_$cfg.err
done
# stress: the settings a P = 8 run would use (16 NVLS CTAs) and the CTA-pair kernel forced on
for i in 1 2 3; do
  for cfg in c3 c1; do
    port=$((port+1))
    POS_NVLS_CTAS=16 POS_SFB_PAIR=1 timeout 300 $T --master-port $port bench.py --gpus $N --steps 30 --warmup 5 --config $cfg --no-cpu-baseline --no-e2e --no-tf32 > $O/stress_${cfg}_$i.json 2> $O/stress_${cfg}_$i.err; echo "stress $cfg $i rc=$?" >> $O/stress.log
  done
done
timeout 600 $T --master-port 29599 scripts/scheme_crossover.py $O/scheme_crossover.json > $O/crossover.log 2>&1; echo "xover rc=$?" >> $O/crossover.log
tail -n 2 $O/pytest_multi.log $O/nvlink.log $O/crossover.log
cat $O/stress.log
for cfg in c3 c1 c2 c4; do python -c "import json; d=json.loads(open('$O/bench_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],4), round(d['roofline']['step']['frac_pipelined'],3), d['clocks'])" 2>&1 | tail -1; done
