"""NVLink traffic of the collective kernels, from the GPUs' own NVLink data counters (NVML field
values NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX / _RX, cumulative KiB over all links): for each method
the bytes one rank sends / receives per synchronisation unit of n fp32 parameters, next to the
algorithmic volume of a reduce-scatter + all-gather, 2 (P-1)/P * 4 n bytes per direction
 — the "traffic" evidence for the fused PS kernels (which ncu cannot replay across
ranks).

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 scripts/nvlink_bytes.py [out.json]
"""
import json
import os
import sys
import time

import pynvml
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
out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", f"nvlink_bytes_p{world}.json")
P = world

pynvml.nvmlInit()


def _nvml_handle():
    """The NVML handle of this rank's CUDA device (matched by UUID; CUDA and NVML orders may differ)."""
    want = str(torch.cuda.get_device_properties(dev).uuid).replace("GPU-", "").lower()
    for i in range(pynvml.nvmlDeviceGetCount()):
        hh = pynvml.nvmlDeviceGetHandleByIndex(i)
        u = pynvml.nvmlDeviceGetUUID(hh)
        u = (u.decode() if isinstance(u, bytes) else u).replace("GPU-", "").lower()
        if u == want:
            return hh
    return pynvml.nvmlDeviceGetHandleByIndex(local)


h = _nvml_handle()


_LINKS = list(range(pynvml.NVML_NVLINK_MAX_LINKS))


def counters():
    """(tx KiB, rx KiB) summed over the links that report (scopeId = link)."""
    q = [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, l) for l in _LINKS] + \
        [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, l) for l in _LINKS]
    vals = pynvml.nvmlDeviceGetFieldValues(h, q)
    if not any(v.nvmlReturn == 0 for v in vals):
        # the round-2 pool reports NOT_SUPPORTED here (nvidia-smi nvlink -gt d: N/A on every link)
        raise RuntimeError("NVLink throughput counters are not supported on this system")
    tx = sum(v.value.ullVal for v in vals[:len(_LINKS)] if v.nvmlReturn == 0)
    rx = sum(v.value.ullVal for v in vals[len(_LINKS):] if v.nvmlReturn == 0)
    return tx, rx


def measure(fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    time.sleep(0.2)
    tx0, rx0 = counters()
    for _ in range(iters):
        fn()
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    time.sleep(1.5)                      # the counters are updated asynchronously
    tx1, rx1 = counters()
    return (tx1 - tx0) * 1024 / iters, (rx1 - rx0) * 1024 / iters


rows = []
iters = 200
for mib in (16, 64):
    n = mib * 2 ** 20 // 4
    n -= n % (64 * P)
    alg = 2 * (P - 1) / P * 4 * n                   # RS + AG, bytes per rank and direction
    Pn = pos.pos_padded_size(n, P)
    Ws, Gs = ctx.sym_empty(Pn), ctx.sym_empty(Pn)
    Gs.normal_()
    res = {"MiB": mib, "n": n, "algorithmic_rs_ag_bytes_per_dir": alg}
    orders = [(pos.POS_REDUCE_SWITCH, "fused_nvls"), (pos.POS_REDUCE_RANK_ORDER, "fused_rank_order")]
    if P == 2:
        orders.append((pos.POS_REDUCE_AUTO, "fused_p2p"))
    for order, name in orders:
        ctx.set_reduce_order(order)
        tx, rx = measure(lambda: ctx.sync_layer_ps(n, Gs, Ws, -1e-9), iters)
        res[name] = {"tx_bytes": tx, "rx_bytes": rx, "tx_over_alg": tx / alg, "rx_over_alg": rx / alg}
    ctx.set_reduce_order(pos.POS_REDUCE_AUTO)
    x = torch.randn(n, device=dev)
    y = torch.empty(n // P, device=dev)
    tx_rs, rx_rs = measure(lambda: dist.reduce_scatter_tensor(y, x), iters)
    tx_ag, rx_ag = measure(lambda: dist.all_gather_into_tensor(x, y), iters)
    res["nccl_rs_plus_ag"] = {"tx_bytes": tx_rs + tx_ag, "rx_bytes": rx_rs + rx_ag,
                              "tx_over_alg": (tx_rs + tx_ag) / alg, "rx_over_alg": (rx_rs + rx_ag) / alg}
    t = torch.tensor([res[k]["tx_bytes"] for k in res if isinstance(res[k], dict)], device=dev, dtype=torch.float64)
    allr = [torch.zeros_like(t) for _ in range(P)]
    dist.all_gather(allr, t)
    res["tx_bytes_all_ranks"] = [a.tolist() for a in allr]
    rows.append(res)
    if rank == 0:
        print(json.dumps(res), flush=True)
    del x, y

if rank == 0:
    with open(out_path, "w") as f:
        json.dump({"P": P, "rows": rows, "gpu": torch.cuda.get_device_name(dev),
                   "how": "NVML NVLINK_THROUGHPUT_DATA_TX/RX deltas (KiB, all links) around 200 units, "
                          "per unit; algorithmic = reduce-scatter + all-gather volume 2 (P-1)/P * 4 n"}, f, indent=1)
dist.barrier(device_ids=[local])
ctx.close()
dist.destroy_process_group()
