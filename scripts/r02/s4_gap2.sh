# 2 GPUs: PS launch gap vs reconstruction stream count / comm priority (c3, c2)
O=gpurun_out/r02/gap2; mkdir -p $O
export POS_TIMEOUT_MS=20000
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
port=29450
for cfg in c3 c2; do
  for v in "POS_SFB_STREAMS=1" "POS_SFB_STREAMS=2" "POS_SFB_STREAMS=3" "POS_PACK_STREAM=1"; do
    port=$((port+1)); tag=$(echo $v | tr '=' '_')
    timeout 300 env $v $T --master-port $port bench.py --gpus $NG --config $cfg --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 > $O/b_${cfg}_${tag}_n${NG}.json 2> $O/b_${cfg}_${tag}_n${NG}.err
    echo "$cfg $v rc=$? $(python -c "
import json; d=json.loads(open('$O/b_${cfg}_${tag}_n${NG}.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4))
for r in sorted(d['trace_timeline_us'], key=lambda r: r[2]): print('   ', r)" 2>&1 | tail -9)"
  done
done
