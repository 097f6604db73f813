N=$(nvidia-smi -L | wc -l)
port=29700
run() {  # label, env...
  port=$((port+1))
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $C --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/o.json 2> gpurun_out/o.err
  echo "N=$N [$C] $LBL $(python scripts/show_bench.py gpurun_out/o.json | cut -c1-120)"
}
for C in c3 c4; do
LBL=default run X=1
LBL=nv16 run POS_NVLS_CTAS=16
LBL=nv64 run POS_NVLS_CTAS=64
LBL=a4_132 run POS_SFB_MAX_CTAS=132
LBL=a4_116 run POS_SFB_MAX_CTAS=116
LBL=a4_116_nv16 run POS_SFB_MAX_CTAS=116 POS_NVLS_CTAS=16
done
