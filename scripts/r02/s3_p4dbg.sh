# 4 GPUs: the P=8 NVLS grid (16 CTAs) on c3 without / with the forced CTA-pair kernel (stress hang of the previous call), with async-error checks; then the exposure measurement at P=4
N=4
O=gpurun_out/r02/p4dbg; mkdir -p $O
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29720
run() { name=$1; shift; port=$((port+1)); timeout 150 env "$@" $T --master-port $port bench.py --gpus $N --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-tf32 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name rc=$? $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['step']['frac_pipelined'],3))" 2>&1 | tail -1)"; }
ARGS="--config c3" run c3_ctas16_a POS_NVLS_CTAS=16 POS_TIMEOUT_MS=5000
ARGS="--config c3" run c3_ctas16_b POS_NVLS_CTAS=16 POS_TIMEOUT_MS=5000
ARGS="--config c3" run c3_pair POS_SFB_PAIR=1 POS_TIMEOUT_MS=5000
ARGS="--config c3" run c3_pair_ctas16 POS_SFB_PAIR=1 POS_NVLS_CTAS=16 POS_TIMEOUT_MS=3000 POS_BENCH_VERBOSE=1
grep -h "PoseidonError\|watchdog\|Error" $O/c3_pair*.err | sort | uniq -c | head -10
bash scripts/r02/s3_wfbp.sh 4
