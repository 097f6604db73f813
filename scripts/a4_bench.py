"""Isolated timing of the A4 reconstruct-and-apply kernel (pos_reconstruct_apply) on the bench
shapes: CUDA events around each launch on its stream, inputs larger than L2 rotated between
launches. Prints algorithmic GB/s (8MN + 2KP(M+N)) and fraction of the measured HBM peak."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
shapes = [(4096, 25088, 32), (21841, 4096, 32), (4096, 4096, 32), (4096, 25088, 256), (21841, 4096, 256), (4096, 9216, 512), (4096, 9216, 1024)]
if os.environ.get("A4_SHAPES"):
    shapes = [tuple(map(int, x.split(","))) for x in os.environ["A4_SHAPES"].split(";")]
tag = os.environ.get("TAG", os.path.basename(pos.LIB_PATH))
for (M, N, KP) in shapes:
    R = pos.pos_factor_row_elems(M, N)
    G = (torch.randn(KP, R, device="cuda") * 0.03).to(torch.bfloat16)
    nrot = 3
    Ws = [torch.randn(M, N, device="cuda") for _ in range(nrot)]
    for i in range(3):
        pos.pos_reconstruct_apply(M, N, KP, pos.POS_DT_BF16, G, Ws[i % nrot], None, -1e-3)
    torch.cuda.synchronize()
    # back-to-back launches between two events: the host-side TMA-descriptor encoding of each call
    # overlaps the previous kernel instead of sitting inside a single-launch event bracket
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for i in range(12):
            pos.pos_reconstruct_apply(M, N, KP, pos.POS_DT_BF16, G, Ws[i % nrot], None, -1e-3)
        e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 12)
    ts.sort(); t = ts[1] * 1e-3
    byts = 8 * M * N + 2 * KP * (M + N)
    print(json.dumps({"tag": tag, "M": M, "N": N, "KP": KP, "us": round(t * 1e6, 1), "GBs": round(byts / t / 1e9), "frac": round(byts / t / 1e9 / peak, 3),
                      "tflops": round(2 * M * N * KP / t / 1e12, 1)}), flush=True)
# streaming reference: A7 shard apply (read g, read W, write W) over 100M elements
n = 100 * 2**20
g = torch.randn(n, device="cuda"); Wx = [torch.randn(n, device="cuda") for _ in range(2)]
for i in range(3): pos.pos_ps_apply(g, Wx[i % 2], n, -1e-3)
torch.cuda.synchronize(); ts = []
for i in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); pos.pos_ps_apply(g, Wx[i % 2], n, -1e-3); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort(); t = ts[5] * 1e-3
print(json.dumps({"tag": tag, "M": 0, "N": n, "KP": 0, "us": round(t * 1e6, 1), "GBs": round(12 * n / t / 1e9), "frac": round(12 * n / t / 1e9 / peak, 3), "tflops": 0}), flush=True)
# copy reference (torch): read + write
for i in range(3): Wx[0].copy_(Wx[1])
torch.cuda.synchronize(); ts = []
for i in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); Wx[i % 2].copy_(Wx[(i + 1) % 2]); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort(); t = ts[5] * 1e-3
print(json.dumps({"tag": tag, "M": 1, "N": n, "KP": 0, "us": round(t * 1e6, 1), "GBs": round(8 * n / t / 1e9), "frac": round(8 * n / t / 1e9 / peak, 3), "tflops": 0}), flush=True)
