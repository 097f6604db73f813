# exposure script at P=1 / P=2 (graph and eager) to locate the P>1 capture failure; multi-GPU tests with the cluster-off default
O=gpurun_out/r02/wfbpdbg; mkdir -p $O
export POS_TIMEOUT_MS=20000
timeout 600 python scripts/wfbp_train_bench.py --config c1 --graph --steps 10 > $O/c1_p1_graph.json 2> $O/c1_p1_graph.err; echo "p1 graph rc=$? $(tail -1 $O/c1_p1_graph.json | cut -c1-300)"
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
TORCH_SHOW_CPP_STACKTRACES=1 WFBP_ONLY=1 timeout 600 $T --master-port 29781 scripts/wfbp_train_bench.py --config c1 --graph --steps 10 > $O/c1_p2_graph.json 2> $O/c1_p2_graph.err; echo "p2 graph rc=$? $(tail -1 $O/c1_p2_graph.json | cut -c1-300)"
WFBP_ONLY=1 timeout 600 $T --master-port 29782 scripts/wfbp_train_bench.py --config c1 --steps 10 > $O/c1_p2_eager.json 2> $O/c1_p2_eager.err; echo "p2 eager rc=$? $(tail -1 $O/c1_p2_eager.json | cut -c1-300)"
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_multi_model.py -x -q > $O/pytest_multi.log 2>&1; echo "multi rc=$?"; tail -2 $O/pytest_multi.log
