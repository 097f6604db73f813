# exposed sync in a real training step (autograd WFBP driver, whole step as one CUDA graph) at N GPUs
N=${1:-1}
O=gpurun_out/r02/wfbp; mkdir -p $O
export POS_TIMEOUT_MS=20000
for cfg in c3 c1 c4; do
  if [ $N = 1 ]; then
    timeout 600 python scripts/wfbp_train_bench.py --config $cfg --graph --steps 20 > $O/${cfg}_p$N.json 2> $O/${cfg}_p$N.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29650 + ${#cfg} + RANDOM % 100)) scripts/wfbp_train_bench.py --config $cfg --graph --steps 20 > $O/${cfg}_p$N.json 2> $O/${cfg}_p$N.err
  fi
  echo "$cfg P=$N rc=$? $(tail -1 $O/${cfg}_p$N.json | cut -c1-400)"
done
