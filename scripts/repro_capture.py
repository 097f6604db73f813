import os, sys, traceback
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local); dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
ctx = pos.Context.from_torch_distributed()
n = 590080
Pn = pos.pos_padded_size(n, world)
for timing in (False, "apply", True):
    for symm in (False, True):
        sch = pos.Scheduler(ctx, 1, timing=timing)
        W = ctx.sym_empty(Pn) if symm else torch.zeros(Pn, device=dev)
        G = ctx.sym_empty(Pn) if symm else torch.zeros(Pn, device=dev)
        sch.add_dense(0, n, W, G)
        def step(s):
            sch.begin(1.0); sch.grad_ready(0, s); sch.end(s)
        try:
            step(torch.cuda.current_stream()); torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph(); cs = torch.cuda.Stream(); cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
                step(torch.cuda.current_stream())
            g.replay(); torch.cuda.synchronize()
            print(f"rank{rank} timing={timing} symm={symm}: OK", flush=True)
        except Exception as e:
            print(f"rank{rank} timing={timing} symm={symm}: FAIL {str(e).splitlines()[0]}", flush=True)
            torch.cuda.synchronize()
        del g
        sch.close()
ctx.close()
dist.destroy_process_group()
