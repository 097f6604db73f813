# N GPUs: two PS lanes on top of the round-2 defaults (epoch barriers, deferred exit, pack placement)
O=gpurun_out/r02/lanes; mkdir -p $O
export POS_TIMEOUT_MS=20000
port=29150
for NG in 4 2; do
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
for cfg in c2 c4 c3; do
  for l in 2 1; do
    port=$((port+1))
    timeout 300 env POS_PS_LANES=$l $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_l${l}_n${NG}.json 2> $O/b_${cfg}_l${l}_n${NG}.err
    echo "P$NG $cfg lanes=$l rc=$? $(python -c "
import json; d=json.loads(open('$O/b_${cfg}_l${l}_n${NG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))" 2>&1 | tail -1)"
  done
done
done
