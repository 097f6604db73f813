"""NEXT-3 validation: for FC layers near the SFB / PS crossover, time the two schemes
end to end at P ranks and compare the winner with Algorithm 1 and with the
B200-calibrated time model (pos_scheme_times_b200).

  SFB: the scheduler's FC unit forced to SFB — fused pack + multicast gather of the factors +
       replicated reconstruct-and-apply (+ bias)
  PS : the same layer forced to PS — G_r = U_r^T V_r formed locally (the dense gradient a PS worker
       pushes) + fused reduce-scatter / shard apply / all-gather of [W | b] (symmetric buffers)

Device time per step (one-layer step captured as CUDA graphs, 20 replays between CUDA events),
median of 3, max over ranks.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 scripts/scheme_crossover.py [out.json]
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
out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", f"scheme_crossover_p{world}.json")
P = world

# (M, N, K): GoogLeNet's FC at the paper's K = 128, the VERDICT's 1000x1024 K = 256,
# Inception-V3's FCs, AlexNet / VGG FCs at their K, and shapes that straddle K* = 2MN / (P(M+N)).
SHAPES = [(1000, 1024, 128), (1000, 1024, 256), (1000, 1024, 512), (1000, 2048, 32), (1000, 768, 32),
          (1000, 768, 256), (4096, 4096, 32), (4096, 4096, 128), (4096, 4096, 512), (1000, 4096, 256),
          (4096, 9216, 128), (2048, 2048, 512)]


def timeit(step, iters=20, reps=3):
    """step(stream) issues one synchronisation; 4 CUDA graphs of one step each are replayed round
    robin (the flag-mode gather alternates buffers by iteration parity)."""
    main = torch.cuda.current_stream()
    for _ in range(3):
        step(main)
    torch.cuda.synchronize()
    gs, cs = [], torch.cuda.Stream()
    cs.wait_stream(main)
    for _ in range(4):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
            step(torch.cuda.current_stream())
        gs.append(g)
    main.wait_stream(cs)
    for g in gs:
        g.replay()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for i in range(iters):
            gs[i % 4].replay()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ts.append(t.item())
    return statistics.median(ts) * 1e3   # us


def one_layer(M, N, K, u, v, scheme):
    """A one-layer scheduler with the scheme forced; returns (step, scheduler)."""
    sch = pos.Scheduler(ctx, 1)
    if scheme == pos.POS_SCHEME_SFB:
        W = torch.randn(M, N, device=dev) * 0.01
        b = torch.zeros(M, device=dev)
        keep = (W, b)
        assert sch.add_fc(0, M, N, K, W, b, None, "bf16", pos.POS_IN_BF16, force_scheme=scheme) == scheme
    else:
        n = M * N + M
        Wb = ctx.sym_empty(pos.pos_padded_size(n, P))
        grad = ctx.sym_empty(pos.pos_padded_size(n, P))
        keep = (Wb, grad)
        assert sch.add_fc(0, M, N, K, Wb[:M * N], Wb[M * N:n], grad, "bf16", pos.POS_IN_BF16,
                          force_scheme=scheme) == scheme

    def step(stream):
        sch.begin(-1e-4)
        sch.factors_ready(0, u, v, stream)
        sch.end(stream)
    return step, sch, keep


rows = []
for (M, N, K) in SHAPES:
    g = torch.Generator(device=dev)
    g.manual_seed(100 + rank)
    u = (torch.randn(K, M, device=dev, generator=g) * 0.03).to(torch.bfloat16)
    v = torch.relu(torch.randn(K, N, device=dev, generator=g)).to(torch.bfloat16)
    t = {}
    for scheme in (pos.POS_SCHEME_SFB, pos.POS_SCHEME_PS):
        step, sch, keep = one_layer(M, N, K, u, v, scheme)
        t[scheme] = timeit(step)
        torch.cuda.synchronize()
        sch.close()
        del keep
    t_sfb, t_ps = t[pos.POS_SCHEME_SFB], t[pos.POS_SCHEME_PS]
    alg1 = pos.SCHEME_NAMES[pos.pos_choose_scheme(M, N, K, P)]
    s_b, m_sfb, m_ps = pos.pos_scheme_times_b200(M, N, K, P)
    row = {"M": M, "N": N, "K": K, "P": P, "t_sfb_us": t_sfb, "t_ps_us": t_ps,
           "measured": "SFB" if t_sfb <= t_ps else "PS", "alg1": alg1,
           "b200_model": pos.SCHEME_NAMES[s_b], "model_sfb_us": m_sfb * 1e6, "model_ps_us": m_ps * 1e6,
           "model_adam_us": pos.pos_scheme_time_adam_b200(M, N, K, P) * 1e6}
    rows.append(row)
    if rank == 0:
        print(json.dumps(row), flush=True)

if rank == 0:
    agree_alg1 = sum(r["measured"] == r["alg1"] for r in rows)
    agree_b200 = sum(r["measured"] == r["b200_model"] for r in rows)
    res = {"P": P, "rows": rows, "agree_alg1": agree_alg1, "agree_b200_model": agree_b200, "n": len(rows),
           "how": "device time per one-layer scheduler step (CUDA-graph replays between CUDA events), median "
                  "of 3, max over ranks; scheme forced per run (add_fc force_scheme); bf16 factors, fp32 W / "
                  "gradients, symmetric (NVLS) buffers",
           "gpu": torch.cuda.get_device_name(dev)}
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as f:
        json.dump(res, f, indent=1)
    print(f"measured winner agrees with Alg. 1 on {agree_alg1}/{len(rows)}, with the B200 model on {agree_b200}/{len(rows)}")
dist.barrier(device_ids=[local])
ctx.close()
dist.destroy_process_group()
