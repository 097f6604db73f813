"""One PS unit alone through the scheduler at P ranks (torchrun): device time per synchronisation of
n fp32 parameters, step graphs replayed back to back, max over ranks — for comparing the PS
transports (POS_PS_CE=1: copy engines; 0: the fused SM kernel) without a co-running
reconstruction. Prints one JSON line per size: ms, and per-direction GB/s of the
reduce-scatter + all-gather volume 2 (P-1)/P * 4n.

    POS_PS_CE=1 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ps_unit_bench.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1706_03292_b200 as pos  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = pos.Context.from_torch_distributed()
P = world
for mib in [int(x) for x in (sys.argv[1:] or ["4", "16", "64", "256"])]:
    n = mib * 2 ** 20 // 4
    Pn = pos.pos_padded_size(n, P)
    W, g = ctx.sym_empty(Pn), ctx.sym_empty(Pn)
    g.normal_()
    W.zero_()
    sch = pos.Scheduler(ctx, 1)
    sch.add_dense(0, n, W, g)

    def step(s):
        sch.begin(-1e-6)
        sch.grad_ready(0, s)
        sch.end(s)

    main = torch.cuda.current_stream()
    for _ in range(3):
        step(main)
    torch.cuda.synchronize()
    cs = torch.cuda.Stream()
    cs.wait_stream(main)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=cs, capture_error_mode="thread_local"):
        step(torch.cuda.current_stream())
    main.wait_stream(cs)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    it = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / it], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    if rank == 0:
        vol = 2 * (P - 1) / P * 4 * n
        print(json.dumps({"MiB": mib, "P": P, "ce": ctx_ce if (ctx_ce := os.environ.get("POS_PS_CE")) else "0",
                          "ms": ms, "gbs_per_dir": vol / ms / 1e6}), flush=True)
    del gr
    sch.close()
    del W, g
ctx.close()
dist.destroy_process_group()
