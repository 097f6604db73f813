# 2 GPUs, clean A/B (no per-stage events): pack stream on/off; bucket size
export POS_TIMEOUT_MS=20000
O=gpurun_out/r02/ab2; mkdir -p $O
NG=${1:-2}
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node ${1:-2} --master-addr 127.0.0.1"
port=29800
run() { name=$1; shift; port=$((port+1)); timeout 300 env "$@" $T --master-port $port bench.py --gpus $NG --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['step']['frac_pipelined'],3))" 2>&1 | tail -1)"; }
for rep in 1 2; do
for cfg in c3 c1 c2 c4; do
  ARGS="--config $cfg" run pk_${cfg}_$rep POS_PACK_STREAM=1
  ARGS="--config $cfg" run nopk_${cfg}_$rep POS_PACK_STREAM=0
done
done
for b in 32 64; do
  ARGS="--config c3 --bucket-mb $b" run pk_c3_b$b POS_PACK_STREAM=1
  ARGS="--config c4 --bucket-mb $b" run pk_c4_b$b POS_PACK_STREAM=1
done
