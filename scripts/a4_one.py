"""One warm A4 launch per shape given on the command line as M,N,KP (for ncu captures)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_03292_b200 as pos
for spec in sys.argv[1:]:
    M, N, KP = map(int, spec.split(","))
    R = pos.pos_factor_row_elems(M, N)
    G = (torch.randn(KP, R, device="cuda") * 0.03).to(torch.bfloat16)
    W = torch.randn(M, N, device="cuda")
    for i in range(2):
        pos.pos_reconstruct_apply(M, N, KP, pos.POS_DT_BF16, G, W, None, -1e-3)
    torch.cuda.synchronize()
    print(spec, "ok", flush=True)
