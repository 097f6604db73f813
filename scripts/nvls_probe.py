"""NVLS fused PS kernel vs NCCL RS+apply+AG (pos_sync_layer_ps) vs torch NCCL RS / AG, by size."""
import json, os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = pos.Context.from_torch_distributed()
def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); dist.barrier(device_ids=[local])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev); dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() * 1e3
tag = os.environ.get("TAG", "")
for mb in [float(x) for x in os.environ.get('PROBE_MB', '4,19,80').split(',')]:
    n = int(mb * 2**20) // 4
    Pn = pos.pos_padded_size(n, world)
    Ws, Gs = ctx.sym_empty(Pn), ctx.sym_empty(Pn)
    Wd, Gd = torch.zeros(Pn, device=dev), torch.zeros(Pn, device=dev)
    t_nvls = timeit(lambda: ctx.sync_layer_ps(n, Gs, Ws, -1e-3))
    t_nccl = timeit(lambda: ctx.sync_layer_ps(n, Gd, Wd, -1e-3))
    y = torch.empty(Pn // world, device=dev)
    t_rs = timeit(lambda: dist.reduce_scatter_tensor(y, Gd))
    t_ag = timeit(lambda: dist.all_gather_into_tensor(Gd, y))
    t_ar = timeit(lambda: dist.all_reduce(Gd))
    # per-rank NVLink bytes per direction of the PS exchange (ring RS + AG): 2 (P-1)/P n 4
    nvl = 2 * (world - 1) / world * n * 4
    if rank == 0:
        print(json.dumps({"tag": tag, "P": world, "MB": mb, "nvls_us": round(t_nvls, 1), "nccl_ps_us": round(t_nccl, 1),
                          "torch_rs_us": round(t_rs, 1), "torch_ag_us": round(t_ag, 1), "torch_allreduce_us": round(t_ar, 1),
                          "nvls_GBs_ringequiv": round(nvl / t_nvls / 1e3), "nccl_GBs": round(nvl / t_nccl / 1e3)}), flush=True)
ctx.close(); dist.destroy_process_group()
