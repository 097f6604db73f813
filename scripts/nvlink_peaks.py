"""Achievable NVLink / NVSwitch bandwidth on this node ("measure the achievable AG/RS
busbw ... record it next to MEASURED_PEAKS"), nccl-tests style: in-place all-gather and
reduce-scatter of fp32 buffers from 1 MiB to 1 GiB (busbw = algbw * (P-1)/P: the bytes each GPU
moves per direction), plus the library's fused PS unit (NVLS switch-order and fixed rank-order
reduce) at the same sizes. Device time, max over ranks, median of 3 repetitions of 20 launches.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 scripts/nvlink_peaks.py [out.json]

Rank 0 merges its result for this P into the JSON file (default profiles/nvlink_peaks.json), which
bench.py reads for the NVLink term of the roofline.
"""
import json
import os
import statistics
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
out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "nvlink_peaks.json")


def timeit(fn, iters=20, reps=3):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts.append(t.item())
    return statistics.median(ts)   # ms


rows = []
for mb in [1, 4, 16, 64, 256, 1024]:
    n = mb * 2 ** 20 // 4
    n -= n % (64 * world)
    x = torch.randn(n, device=dev)
    y = torch.empty(n // world, device=dev)
    t_ag = timeit(lambda: dist.all_gather_into_tensor(x, y))
    t_rs = timeit(lambda: dist.reduce_scatter_tensor(y, x))
    bus = lambda t: (world - 1) / world * n * 4 / (t * 1e-3) / 1e9
    row = {"MiB": mb, "ag_ms": t_ag, "ag_busbw_gbs": bus(t_ag), "rs_ms": t_rs, "rs_busbw_gbs": bus(t_rs)}
    del x, y
    if mb <= 256:
        Pn = pos.pos_padded_size(n, world)
        Ws, Gs = ctx.sym_empty(Pn), ctx.sym_empty(Pn)
        Gs.normal_()
        orders = [(pos.POS_REDUCE_SWITCH, "nvls"), (pos.POS_REDUCE_RANK_ORDER, "rank_order")]
        if world == 2:
            orders.append((pos.POS_REDUCE_AUTO, "p2p"))   # peer loads + peer stores
        for order, name in orders:
            ctx.set_reduce_order(order)
            t = timeit(lambda: ctx.sync_layer_ps(n, Gs, Ws, -1e-6))
            # a PS unit = reduce-scatter + all-gather volume: 2 (P-1)/P n 4 bytes per direction
            row[f"ps_{name}_ms"] = t
            row[f"ps_{name}_busbw_gbs"] = 2 * bus(t)
        ctx.set_reduce_order(pos.POS_REDUCE_AUTO)
    rows.append(row)
    if rank == 0:
        print(json.dumps(row), flush=True)

if rank == 0:
    res = {}
    if os.path.exists(out_path):
        with open(out_path) as f:
            res = json.load(f)
    res[f"P{world}"] = {
        "ag_busbw_gbs": max(r["ag_busbw_gbs"] for r in rows),
        "rs_busbw_gbs": max(r["rs_busbw_gbs"] for r in rows),
        # the best per-direction rate any method reached: NCCL AG / RS or the fused PS unit
        "per_dir_gbs": max(max(r["ag_busbw_gbs"], r["rs_busbw_gbs"], r.get("ps_nvls_busbw_gbs", 0),
                               r.get("ps_p2p_busbw_gbs", 0)) for r in rows),
        "ps_p2p_busbw_gbs": max(r.get("ps_p2p_busbw_gbs", 0) for r in rows),
        "ps_nvls_busbw_gbs": max(r.get("ps_nvls_busbw_gbs", 0) for r in rows),
        "ps_rank_order_busbw_gbs": max(r.get("ps_rank_order_busbw_gbs", 0) for r in rows),
        "sizes": rows,
        "how": "nccl-tests style in-place AG / RS fp32 (torch.distributed, NCCL " +
               ".".join(map(str, torch.cuda.nccl.version())) + "), device time max over ranks, "
               "median of 3 x 20 launches; busbw = algbw (P-1)/P; per_dir_gbs = max(NCCL AG, NCCL RS, the fused PS unit's RS+AG-equivalent busbw)",
        "gpu": torch.cuda.get_device_name(dev),
    }
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
dist.barrier(device_ids=[local])
ctx.close()
dist.destroy_process_group()
