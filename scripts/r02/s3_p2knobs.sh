# 2 GPUs: defaults vs P2P PS kernel, bucket size and pack stream (clean lines, no per-stage events)
export POS_TIMEOUT_MS=20000
O=gpurun_out/r02/p2knobs; mkdir -p $O
NG=2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
port=29840
run() { name=$1; shift; port=$((port+1)); timeout 300 env "$@" $T --master-port $port bench.py --gpus $NG --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['step_stats']['median_ms'],4), round(d['roofline']['step']['frac_pipelined'],3))" 2>&1 | tail -1)"; }
for cfg in c3 c1 c2 c4; do
  ARGS="--config $cfg" run def_$cfg X=1
  ARGS="--config $cfg" run p2p_$cfg POS_PS_P2P=1
  ARGS="--config $cfg --bucket-mb 64" run b64_$cfg X=1
  ARGS="--config $cfg --bucket-mb 64" run b64pk_$cfg POS_PACK_STREAM=1
  ARGS="--config $cfg --bucket-mb 64" run b64p2p_$cfg POS_PS_P2P=1
done
