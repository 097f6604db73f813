# N GPUs (N = $1): bench line per config (+ per-unit table for c3); TAG = $2
N=${1:-2}; TAG=${2:-pb}
O=gpurun_out/r02/$TAG$N
mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29620
for cfg in c3 c1 c2 c4; do
  port=$((port+1))
  timeout 400 $T --master-port $port bench.py --gpus $N --steps 50 --warmup 10 --config $cfg --layers --no-cpu-baseline --no-e2e --no-tf32 > $O/bench_$cfg.json 2> $O/bench_$cfg.err; echo "bench $cfg rc=$?" >> $O/bench_$cfg.err
done
for cfg in c3 c1 c2 c4; do python -c "import json; d=json.loads(open('$O/bench_$cfg.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],4), round(d['roofline']['step']['frac_pipelined'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
grep -v "^\[" $O/bench_c3.err | tail -9
