"""Per-stage timing of ONE SFB unit (VGG19-22K fc8, K=32) through the scheduler at P ranks: pack
(multicast + barriers) vs reconstruct-and-apply, no other traffic. Rank 0 prints JSON."""
import json, os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = pos.Context.from_torch_distributed()
res = {}
for symm in (True, False):
    for (M, N) in [(21841, 4096), (4096, 4096)]:
        K = 32
        sch = pos.Scheduler(ctx, 1, timing=True, symm=symm)
        W = torch.randn(M, N, device=dev); b = torch.zeros(M, device=dev)
        u = (torch.randn(K, M, device=dev) * 0.03).bfloat16(); v = torch.relu(torch.randn(K, N, device=dev)).bfloat16()
        sch.add_fc(0, M, N, K, W, b, None, "bf16", pos.POS_IN_BF16)
        s = torch.cuda.current_stream()
        for i in range(30):
            if i == 10:
                torch.cuda.synchronize(); sch.timing_reset()
            dist.barrier(device_ids=[local])
            sch.begin(-1e-3); sch.factors_ready(0, u, v, s); sch.end(s)
        torch.cuda.synchronize()
        pk, cm, ap = sch.timing(0)
        res[f"{'nvls' if symm else 'nccl'}_{M}x{N}"] = {"pack_us": round(pk * 1e3, 1), "comm_us": round(cm * 1e3, 1), "apply_us": round(ap * 1e3, 1)}
        sch.close()
if rank == 0:
    print(json.dumps({"P": world, **res}), flush=True)
ctx.close(); dist.destroy_process_group()
