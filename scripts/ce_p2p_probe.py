"""Copy-engine peer bandwidth probe (one process, 2 GPUs): device-to-device copies between GPU 0
and GPU 1 through cudaMemcpyPeerAsync (torch cross-device copy_), one direction and both directions
at once, timed with CUDA events. Context for the NVLink roofline term: the SM-driven fused PS
kernels and NCCL reach ~420-450 GB/s per direction at P = 2 (profiles/nvlink_peaks.json)."""
import json
import sys

import torch

assert torch.cuda.device_count() >= 2
d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
out = {}
for mib in (16, 64, 256, 1024):
    n = mib * 2 ** 20 // 4
    a0, b0 = torch.randn(n, device=d0), torch.empty(n, device=d0)
    a1, b1 = torch.randn(n, device=d1), torch.empty(n, device=d1)
    s0 = torch.cuda.Stream(d0)
    s1 = torch.cuda.Stream(d1)
    res = {}
    for mode in ("uni", "bi"):
        for _ in range(3):
            with torch.cuda.stream(s0):
                b1.copy_(a0, non_blocking=True)
            if mode == "bi":
                with torch.cuda.stream(s1):
                    b0.copy_(a1, non_blocking=True)
        torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
        it = 10
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        f0 = torch.cuda.Event(enable_timing=True); f1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(d0):
            e0.record(s0)
        with torch.cuda.device(d1):
            f0.record(s1)
        for _ in range(it):
            with torch.cuda.stream(s0):
                b1.copy_(a0, non_blocking=True)
            if mode == "bi":
                with torch.cuda.stream(s1):
                    b0.copy_(a1, non_blocking=True)
        with torch.cuda.device(d0):
            e1.record(s0)
        with torch.cuda.device(d1):
            f1.record(s1)
        torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
        ms = e0.elapsed_time(e1) / it
        res[mode + "_gbs_per_dir"] = 4 * n / ms / 1e6
        if mode == "bi":
            res["bi_gbs_dir2"] = 4 * n / (f0.elapsed_time(f1) / it) / 1e6
    out[mib] = res
    print(mib, json.dumps(res), flush=True)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
