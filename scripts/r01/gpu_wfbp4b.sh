N=$(nvidia-smi -L | wc -l)
show() { grep metric $1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('local %.3f nosync %.3f wfbp %.3f seq %.3f exposed_vs_local %.3f (%.3f) vs_nosync %.3f (%.3f)' % (d['ms_step_local_sgd'], d['ms_step_nosync'], d['ms_step_wfbp'], d['ms_step_sequential'], d['exposed_ms_wfbp_vs_local'], d['exposed_frac_wfbp_vs_local'], d['exposed_ms_wfbp'], d['exposed_frac_wfbp']))"; }
for c in c3 c1 c4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29801 scripts/wfbp_train_bench.py --config $c --steps 20 --graph > gpurun_out/wfbp_${c}_n${N}_graph.json 2> gpurun_out/w.err
echo "[$c N=$N graph] $(show gpurun_out/wfbp_${c}_n${N}_graph.json)"
tail -2 gpurun_out/w.err | grep -i error
done
