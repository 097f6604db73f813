# pair-kernel stage/W-slot variants at large K*P (GPU 0), then P=2 comm-stream priority A/B
export POS_TIMEOUT_MS=20000
O=gpurun_out/r02/combo2; mkdir -p $O
export A4_SHAPES="4096,9216,1024;4096,4096,1024;1000,4096,1024;4096,9216,2048"
for v in base ps5pw4 ps6pw2 ps5pw3 ps5pw4e2 ps4pw4 base2; do
  lib=build/libposeidon_$v.so; case $v in base*) lib=paper_1706_03292_b200/libposeidon.so;; esac
  POS_LIB=$PWD/$lib POS_SFB_PAIR=1 TAG=$v timeout 200 python scripts/a4_bench.py 2>&1 | grep "^{" | grep -v '"M": [01],' >> $O/a4.txt
done
python - <<'P'
import json
for l in open("gpurun_out/r02/combo2/a4.txt"):
    d=json.loads(l); print(f"{d['tag']:9s} {d['M']:6d} {d['N']:6d} {d['KP']:5d} {d['us']:7.1f} us  frac_hbm {d['frac']:.3f}  {d['tflops']:7.1f} TF/s")
P
NG=2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1"
port=29900
run() { name=$1; shift; port=$((port+1)); timeout 300 env "$@" $T --master-port $port bench.py --gpus $NG --steps 50 --warmup 10 --no-cpu-baseline --no-e2e --no-tf32 $ARGS > $O/$name.json 2> $O/$name.err; echo "$name $(python -c "import json; d=json.loads(open('$O/$name.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), round(d['roofline']['step']['frac_pipelined'],3))" 2>&1 | tail -1)"; }
for cfg in c3 c1 c2 c4; do
  ARGS="--config $cfg" run nopk_$cfg POS_PACK_STREAM=0
  ARGS="--config $cfg" run pk_p0_$cfg POS_PACK_STREAM=1 POS_COMM_PRIO=0
  ARGS="--config $cfg" run pk_p3_$cfg POS_PACK_STREAM=1 POS_COMM_PRIO=3
  ARGS="--config $cfg" run nopk_p0_$cfg POS_PACK_STREAM=0 POS_COMM_PRIO=0
done
