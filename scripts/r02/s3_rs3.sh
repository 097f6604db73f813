# reconstruction streams 2 vs 3 at P = 1 and P = 2 (timelines)
O=gpurun_out/r02/rs3; mkdir -p $O
export POS_TIMEOUT_MS=20000
for rep in 1 2; do for cfg in c1 c3 c2 c4; do for n in 2 3; do
  POS_SFB_STREAMS=$n timeout 300 python bench.py --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/p1_${cfg}_s$n.json 2>/dev/null
  echo "P1 $cfg s$n $(python -c "import json; d=json.loads(open('$O/p1_${cfg}_s$n.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), [t for t in d['trace_timeline_us'] if t[1]=='SFB'])")"
done; done; done
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
port=29970
for cfg in c3 c1; do for n in 2 3; do port=$((port+1))
  POS_SFB_STREAMS=$n timeout 300 $T --master-port $port bench.py --gpus 2 --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/p2_${cfg}_s$n.json 2>/dev/null
  echo "P2 $cfg s$n $(python -c "import json; d=json.loads(open('$O/p2_${cfg}_s$n.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), [t for t in d['trace_timeline_us'] if t[1]=='SFB'])")"
done; done
