# 4-GPU box: the 1-GPU -m gpu suite + smoke on the final build, then repeated default bench runs at P = 2 and 4 (hang / watchdog check)
O=gpurun_out/r02/stress; mkdir -p $O
export POS_TIMEOUT_MS=20000
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_n1.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_n1.log; tail -2 $O/pytest_gpu_n1.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -1 $O/smoke.log
port=30100
for N in 4 2; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
  for i in 1 2 3 4 5 6; do for cfg in c3 c1; do port=$((port+1))
    timeout 240 $T --master-port $port bench.py --gpus $N --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-tf32 > $O/p${N}_${cfg}_$i.json 2> $O/p${N}_${cfg}_$i.err
    echo "P$N $cfg run $i rc=$? $(python -c "import json; d=json.loads(open('$O/p${N}_${cfg}_$i.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4))" 2>&1 | tail -1)" >> $O/stress.log
  done; done
done
cat $O/stress.log | awk '{print $1, $2, $5, $6}' | sort | uniq -c | sort -rn | head; grep -c "rc=0" $O/stress.log; wc -l < $O/stress.log
