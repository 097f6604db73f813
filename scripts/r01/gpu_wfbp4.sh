N=$(nvidia-smi -L | wc -l)
timeout 300 python -m pytest tests/test_gpu_torch_wfbp.py -q -x 2>&1 | tail -2
for c in c4 c3 c1; do
for g in "" "--graph"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29801 scripts/wfbp_train_bench.py --config $c --steps 20 $g > gpurun_out/wfbp_${c}_n$N$g.json 2> gpurun_out/wfbp_${c}_n$N$g.err
echo "[$c N=$N $g] $(grep metric gpurun_out/wfbp_${c}_n$N$g.json | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('nosync %.3f wfbp %.3f seq %.3f exposed %.3f (%.3f) seq-exposed %.3f' % (d['ms_step_nosync'], d['ms_step_wfbp'], d['ms_step_sequential'], d['exposed_ms_wfbp'], d['exposed_frac_wfbp'], d['exposed_frac_sequential']))")"
tail -3 gpurun_out/wfbp_${c}_n$N$g.err | grep -i "error\|Traceback" 
done; done
