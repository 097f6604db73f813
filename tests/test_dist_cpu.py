"""World-size-2 CPU tests (torch.distributed, gloo) of the N > 1 host logic — no GPU needed.

* the PS shard table drives a distributed reduce-scatter / apply / all-gather played with gloo
  collectives: every rank's result equals the oracle computed from both ranks' gradients, bitwise
  (exact regime), and the shards exchanged are exactly the library's pos_shard_range;
* the SFB gather layout: rank-major slots of K rows of pos_factor_row_elems(M, N) elements, all-gathered
  with gloo, reproduce the oracle's U^T V when contracted on the host;
* the NCCL unique id produced by the library on rank 0 reaches every rank unchanged;
* bench.py's per-rank unit plan / accounting is identical on both ranks and its max-over-ranks
  timing reduction picks the slowest rank.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, outdir, fn_name):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        globals()[fn_name](rank, world)
        open(os.path.join(outdir, f"ok{rank}"), "w").close()
    except Exception:
        import traceback
        open(os.path.join(outdir, f"err{rank}"), "w").write(traceback.format_exc())
    finally:
        dist.destroy_process_group()


def _spawn(fn_name, world=2):
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_run, args=(world, _port(), d, fn_name), nprocs=world, join=True, start_method="spawn")
        errs = [open(os.path.join(d, f)).read() for f in os.listdir(d) if f.startswith("err")]
        assert not errs, errs[0]
        assert len([f for f in os.listdir(d) if f.startswith("ok")]) == world


# ------------------------------------------------------------------------------ workers ------
def _ps_worker(rank, world):
    import paper_1706_03292_b200 as pos
    import synth_inputs as si
    from oracle import sync
    for n in (1, 10, 4097, 2359808):
        g_local = si.exact_dense_grad(si.rng(50, n % 97, rank), n)
        w0 = si.exact_weights(si.rng(50, 1), n)
        a = si.EXACT_ALPHA
        S = pos.pos_shard_stride(n, world)
        buf = np.zeros(world * S, np.float32)
        buf[:n] = g_local
        # reduce-scatter (played with all_gather + local sum of my shard, rank order)
        parts = [torch.zeros(world * S) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(buf))
        lo, hi = pos.pos_shard_range(n, world, rank)
        ghat = sum(p.numpy()[lo:hi].astype(np.float64) for p in parts)
        w = np.zeros(world * S, np.float32)
        w[:n] = w0
        w_shard = np.zeros(S, np.float32)
        w_shard[:hi - lo] = (w[lo:hi].astype(np.float64) + a * ghat).astype(np.float32)
        shards = [torch.zeros(S) for _ in range(world)]
        dist.all_gather(shards, torch.from_numpy(w_shard))
        full = np.concatenate([s.numpy() for s in shards])[:n]
        grads = [si.exact_dense_grad(si.rng(50, n % 97, p), n) for p in range(world)]
        assert np.array_equal(full.astype(np.float64), sync.ps_update(w0, grads, a)), n


def _sfb_worker(rank, world):
    import paper_1706_03292_b200 as pos
    import synth_inputs as si
    from oracle import sync
    K, M, N = 4, 13, 7
    R = pos.pos_factor_row_elems(M, N)
    Mp = (M + 63) // 64 * 64
    u, v = si.exact_factors(si.rng(51, 0, rank), K, M, N)
    slot = np.zeros((K, R), np.float32)
    slot[:, :M] = u
    slot[:, Mp:Mp + N] = v
    slot[:, Mp + N] = 1.0          # the ones column of the ABI layout (bias gradient column)
    gathered = [torch.zeros(K, R) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(slot))
    G = np.concatenate([g.numpy() for g in gathered])          # rows j = p*K + k
    U, V = G[:, :M].astype(np.float64), G[:, Mp:Mp + N].astype(np.float64)
    Us, Vs = zip(*(si.exact_factors(si.rng(51, 0, p), K, M, N) for p in range(world)))
    W0 = si.exact_weights(si.rng(51, 1), M, N)
    ref, _ = sync.sfb_update(W0, None, Us, Vs, si.EXACT_ALPHA)
    assert np.array_equal(W0 + si.EXACT_ALPHA * (U.T @ V), ref)
    # the ones column turns the same contraction into the bias gradient: (U^T 1)[m] = sum_j u_j[m]
    ones = G[:, Mp + N].astype(np.float64)
    assert np.array_equal(U.T @ ones, np.sum(np.concatenate(Us).astype(np.float64), axis=0))
    assert not np.any(G[:, M:Mp]) and not np.any(G[:, Mp + N + 1:])   # other pads stay zero


def _uid_worker(rank, world):
    import paper_1706_03292_b200 as pos
    import ctypes
    buf = ctypes.create_string_buffer(128)
    if rank == 0:
        assert pos.lib().pos_get_unique_id(buf) == 0
    t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone()
    dist.broadcast(t, src=0)
    got = [torch.zeros(128, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(got, t)
    assert all(torch.equal(got[0], g) for g in got) and int(got[0].sum()) > 0


def _bench_worker(rank, world):
    import bench
    import synth_inputs as si
    model = si.load_model("vgg19_22k")
    units = bench.plan_units(model, int(bench.default_bucket_mb(world) * 2 ** 20 / 4))
    rows = bench.unit_accounting(model, units, 32, world, "bf16")
    blob = repr([(r["name"], r["params"], r["hbm_a4"], r["nvl"]) for r in rows]).encode()
    t = torch.tensor(list(blob[:4096]) + [0] * (4096 - len(blob[:4096])), dtype=torch.int64)
    got = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(got, t)
    assert all(torch.equal(got[0], g) for g in got)
    assert sum(u["n"] for u in units) == model.total_params
    ms = torch.tensor([1.0 + rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    assert ms.item() == float(world)


@pytest.mark.parametrize("fn", ["_ps_worker", "_sfb_worker", "_uid_worker", "_bench_worker"])
def test_world2_gloo(fn):
    _spawn(fn)
