# 4 GPUs: repeated default bench runs at P = 4 after kernel preloading
O=gpurun_out/r02/stress2; mkdir -p $O
export POS_TIMEOUT_MS=20000
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
port=30200
for i in $(seq 1 14); do for cfg in c3; do port=$((port+1))
  timeout 200 $T --master-port $port bench.py --gpus 4 --config $cfg --steps 20 --warmup 4 --no-cpu-baseline --no-e2e --no-tf32 > $O/p4_${cfg}_$i.json 2> $O/p4_${cfg}_$i.err
  echo "P4 $cfg run $i rc=$? $(python -c "import json; d=json.loads(open('$O/p4_${cfg}_$i.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))" 2>&1 | tail -1)" >> $O/stress.log
done; done
cat $O/stress.log; grep -c "rc=0" $O/stress.log
