"""NCCL bandwidth probe (nccl-tests style) for the collective shapes of the hot path: in-place
reduce-scatter and all-gather of fp32 buffers, and our own libposeidon PS / SFB syncs in isolation.
Run under torchrun; rank 0 prints one line per size."""
import os, sys, time, json
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = pos.Context.from_torch_distributed()
out = []
def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); dist.barrier(device_ids=[local])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()
for mb in [1, 4, 16, 64, 256]:
    n = mb * 2**20 // 4
    n -= n % (64 * world)
    x = torch.randn(n, device=dev)
    y = torch.empty(n // world, device=dev)
    t_rs = timeit(lambda: dist.reduce_scatter_tensor(y, x))
    t_ag = timeit(lambda: dist.all_gather_into_tensor(x, y))
    W = torch.zeros(pos.pos_padded_size(n, world), device=dev); g = torch.zeros_like(W)
    t_ps = timeit(lambda: ctx.sync_layer_ps(n, g, W, -1e-3))
    bus = lambda t: (world - 1) / world * n * 4 / (t * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({"MB": mb, "torch_rs_ms": t_rs, "rs_busbw": bus(t_rs), "torch_ag_ms": t_ag, "ag_busbw": bus(t_ag),
                          "pos_ps_ms": t_ps, "pos_ps_busbw_rs+ag": 2 * bus(t_ps)}), flush=True)
ctx.close()
dist.destroy_process_group()
