"""Small-shape run of every hot-path kernel for compute-sanitizer (memcheck / racecheck / synccheck):
pack, tensor-core reconstruct-and-apply (bf16 + tf32, ragged tiles), SIMT f32 path, bias, PS apply,
sim PS, and a scheduler iteration (WFBP). Exits non-zero on any mismatch with the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos
import synth_inputs as si
from oracle import sync

def up(x, dt=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda().to(dt)

ok = True
ctx = pos.Context.local_sim(2)
for (M, N, K, dtype) in [(129, 260, 8, "bf16"), (65, 36, 8, "tf32"), (33, 7, 4, "f32"), (300, 520, 32, "bf16")]:
    Us, Vs = zip(*(si.exact_factors(si.rng(1, 0, p), K, M, N) for p in range(2)))
    W, b = si.exact_weights(si.rng(2), M, N), si.exact_weights(si.rng(3), M)
    st = torch.bfloat16 if dtype == "bf16" else torch.float32
    Wd, bd = up(W), up(b)
    ctx.sim_sync_layer_sfb([up(u, st) for u in Us], [up(v, st) for v in Vs], Wd, bd, si.EXACT_ALPHA, dtype)
    torch.cuda.synchronize()
    Wr, br = sync.sfb_update(W, b, Us, Vs, si.EXACT_ALPHA)
    ok &= np.array_equal(Wd.cpu().numpy().astype(np.float64), Wr) and np.array_equal(bd.cpu().numpy().astype(np.float64), br)
n = 1001
gs = [si.exact_dense_grad(si.rng(4, 0, p), n) for p in range(2)]
w = si.exact_weights(si.rng(5), n)
Wd = up(w)
ctx.sim_sync_layer_ps([up(g) for g in gs], Wd, si.EXACT_ALPHA)
torch.cuda.synchronize()
ok &= np.array_equal(Wd.cpu().numpy().astype(np.float64), sync.ps_update(w, gs, si.EXACT_ALPHA))
g1 = up(gs[0]); w1 = up(w)
pos.pos_ps_apply(g1[1:], w1[1:], n - 1, 0.5)   # unaligned scalar path
torch.cuda.synchronize()
# scheduler iteration, world 1 (dynamic tiles, aux-stream pack)
c1 = pos.Context.from_unique_id(bytes(128), 1, 0)
sch = pos.Scheduler(c1, 2, timing=True)
M, N, K = 300, 520, 16
u, v = si.exact_factors(si.rng(6), K, M, N)
W, b = si.exact_weights(si.rng(7), M, N), si.exact_weights(si.rng(8), M)
Wd, bd = up(W), up(b)
sch.add_fc(1, M, N, K, Wd, bd, None, "bf16", pos.POS_IN_BF16)
nd = 777
Pn = pos.pos_padded_size(nd, 1)
Wn = torch.zeros(Pn, device="cuda"); Gn = torch.zeros(Pn, device="cuda")
wn, gn = si.exact_weights(si.rng(9), nd), si.exact_dense_grad(si.rng(10), nd)
Wn[:nd] = up(wn); Gn[:nd] = up(gn)
sch.add_dense(0, nd, Wn, Gn)
ud, vd = up(u, torch.bfloat16), up(v, torch.bfloat16)
for it in range(2):
    sch.begin(si.EXACT_ALPHA); sch.factors_ready(1, ud, vd); sch.grad_ready(0); sch.end()
torch.cuda.synchronize()
W1, b1 = sync.sfb_update(W, b, [u], [v], si.EXACT_ALPHA)
W2, b2 = sync.sfb_update(W1, b1, [u], [v], si.EXACT_ALPHA)
ok &= np.array_equal(Wd.cpu().numpy().astype(np.float64), W2) and np.array_equal(bd.cpu().numpy().astype(np.float64), b2)
ok &= np.array_equal(Wn[:nd].cpu().numpy().astype(np.float64), sync.ps_update(sync.ps_update(wn, [gn], si.EXACT_ALPHA), [gn], si.EXACT_ALPHA))
sch.timing(1)
sch.close(); c1.close(); ctx.close()
# loopback: the P > 1 kernel bodies (flag-mode pack + multicast-slot stores through the pointer
# table, ready flags, flag wait, double-buffered reconstruction; fused shard reduce / apply /
# broadcast) on P = 3 local replicas, two iterations
P = 3
lc = pos.Context.local_sim(P)
M, N, K = 130, 264, 8
Us, Vs = zip(*(si.exact_factors(si.rng(11, 0, p), K, M, N) for p in range(P)))
W, b = si.exact_weights(si.rng(12), M, N), si.exact_weights(si.rng(13), M)
Ws, bs = [up(W) for _ in range(P)], [up(b) for _ in range(P)]
lf = pos.LoopFC(lc, M, N, K, Ws, bs, "bf16")
for it in range(2):
    lf.sync([up(u, torch.bfloat16) for u in Us], [up(v, torch.bfloat16) for v in Vs], si.EXACT_ALPHA)
torch.cuda.synchronize()
Wr, br = W, b
for it in range(2):
    Wr, br = sync.sfb_update(Wr, br, Us, Vs, si.EXACT_ALPHA)
ok &= all(np.array_equal(x.cpu().numpy().astype(np.float64), Wr) for x in Ws)
ok &= all(np.array_equal(x.cpu().numpy().astype(np.float64), br) for x in bs)
lf.close()
n = 3001
Pn = pos.pos_padded_size(n, P)
gs = [si.exact_dense_grad(si.rng(14, 0, p), n) for p in range(P)]
w = si.exact_weights(si.rng(15), n)
Gd = [torch.zeros(Pn, device="cuda") for _ in range(P)]
Wd = [torch.zeros(Pn, device="cuda") for _ in range(P)]
for p in range(P):
    Gd[p][:n] = up(gs[p]); Wd[p][:n] = up(w)
lc.loop_sync_layer_ps(n, Gd, Wd, si.EXACT_ALPHA)
torch.cuda.synchronize()
ref = sync.ps_update(w, gs, si.EXACT_ALPHA)
ok &= all(np.array_equal(x[:n].cpu().numpy().astype(np.float64), ref) for x in Wd)
lc.close()
# CTA-pair (cluster) reconstruction on a ragged shape
os.environ["POS_SFB_PAIR"] = "1"
c2 = pos.Context.local_sim(2)
M, N, K = 257, 132, 8
Us, Vs = zip(*(si.exact_factors(si.rng(16, 0, p), K, M, N) for p in range(2)))
W, b = si.exact_weights(si.rng(17), M, N), si.exact_weights(si.rng(18), M)
Wd, bd = up(W), up(b)
c2.sim_sync_layer_sfb([up(u, torch.bfloat16) for u in Us], [up(v, torch.bfloat16) for v in Vs], Wd, bd, si.EXACT_ALPHA, "bf16")
torch.cuda.synchronize()
Wr, br = sync.sfb_update(W, b, Us, Vs, si.EXACT_ALPHA)
ok &= np.array_equal(Wd.cpu().numpy().astype(np.float64), Wr) and np.array_equal(bd.cpu().numpy().astype(np.float64), br)
c2.close()
print("sanitize_small:", "OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
