"""Multi-GPU (>= 2 B200 of one node) north-star checks, one process per GPU:

* the full VGG19-22K model: bench.py's own step (plan_units, register_units with
  symmetric buffers, make_step, capture_ring) on every rank, fed each rank's host-generated exact
  inputs; rank 0 compares every layer with the oracle summing ALL ranks' inputs (Eq. 2), all ranks
  compare digests (replicas bitwise identical);
* run-to-run determinism of the PS reduce (NEXT-1): the fixed RANK-ORDER reduce is bitwise
  reproducible (asserted); the switch (NVLS) order is recorded;
* grids that differ per rank are impossible (n = 16400 at P = 2);
* the watchdog: a rank that never joins a PS unit (injected fault) makes its peers' barrier time out
  with POS_ETIMEOUT instead of hanging.
"""
import hashlib
import json
import os
import socket
import tempfile

import numpy as np
import pytest

from tests._util import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpu():
    if not have_gpu():
        return 0
    import torch
    return torch.cuda.device_count()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _digest(t) -> str:
    return hashlib.sha256(t.detach().cpu().numpy().tobytes()).hexdigest()


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    import bench
    import paper_1706_03292_b200 as pos
    import synth_inputs as si
    from oracle import sync
    from tests._util import err, to_dev, to_host
    from tests.test_gpu_fullmodel import HostFill, oracle_model

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    res = {"rank": rank, "checks": {}, "digests": {}, "info": {}}
    P = world

    def check(name, ok):
        res["checks"][name] = bool(ok)

    try:
        ctx = pos.Context.from_torch_distributed()
        # ---- (a) full VGG19-22K, bench step, graph ring, exact regime ----------------------------
        def full_model(ctx, key):
            model_name, K = si.CONFIGS["c3"]
            model = si.load_model(model_name)
            units = bench.plan_units(model, int(bench.default_bucket_mb(P) * 2 ** 20 / 4))
            sch = pos.Scheduler(ctx, len(model.layers), timing="apply")
            fill = HostFill("exact", K, rank=rank)
            bufs = bench.register_units(pos, ctx, sch, model, units, K, "bf16", fill)
            a = si.EXACT_ALPHA
            main = torch.cuda.current_stream()
            step = bench.make_step(sch, bufs, a)
            torch.cuda.synchronize()
            dist.barrier(device_ids=[rank])
            for _ in range(3):
                step(main)
            ring = bench.capture_ring(step, main)
            for g in ring:
                g.replay()
            n_iter = 3 + len(ring)
            torch.cuda.synchronize()
            res["digests"][key] = "".join(_digest(bb["W"]) for bb in bufs)
            if rank == 0:
                others = []
                for q in range(1, P):
                    o = {}
                    for l, ly in enumerate(model.layers):
                        if ly.kind == "fc":
                            o[(l, "u")] = fill.value("fc", l, (K, ly.M), "u", q)
                            o[(l, "v")] = fill.value("fc", l, (K, ly.N), "v", q)
                        else:
                            o[(l, "g")] = fill.value("dense", l, (ly.n,), "g", q)
                    others.append(o)
                ref = oracle_model(model, fill.host, n_iter, a, others)
                bad = []
                for l, ly in enumerate(model.layers):
                    got = to_host(bufs[l]["W"]).reshape(ref[l][0].shape)
                    if not np.array_equal(got, ref[l][0]):
                        bad.append(ly.name)
                    if ref[l][1] is not None and not np.array_equal(to_host(bufs[l]["b"]), ref[l][1]):
                        bad.append(ly.name + ".bias")
                res["info"][key + "_bad_layers"] = bad
                check(key + "_graph_ring_exact_oracle", not bad)
            ring = None
            sch.close()
        full_model(ctx, "vgg19_22k")
        # the same with the fused PS units on two lanes (own streams and barrier epochs)
        os.environ["POS_PS_LANES"] = "2"
        try:
            ctx_l = pos.Context.from_torch_distributed()
        finally:
            del os.environ["POS_PS_LANES"]
        full_model(ctx_l, "vgg19_22k_lanes2")
        ctx_l.close()
        # the same with the PS units on the copy engines (POS_PS_CE: pushes + flags + local apply)
        os.environ["POS_PS_CE"] = "1"
        try:
            ctx_ce = pos.Context.from_torch_distributed()
        finally:
            del os.environ["POS_PS_CE"]
        full_model(ctx_ce, "vgg19_22k_ce")
        ctx_ce.close()

        # ---- (b) PS determinism: switch order (recorded) and rank order (asserted) ----------------
        n = 2359808 * 4 + 4097
        Pn = pos.pos_padded_size(n, P)
        gl = si.stat_dense_grad(si.rng(95, 0, rank), n)
        w0 = si.stat_weights(si.rng(96), 1, n)[0]
        Ws, Gs = ctx.sym_empty(Pn), ctx.sym_empty(Pn)
        Gs[:n] = to_dev(gl)
        for order, name in ((pos.POS_REDUCE_SWITCH, "switch"), (pos.POS_REDUCE_RANK_ORDER, "rank_order"),
                            (pos.POS_REDUCE_AUTO, "auto")):
            ctx.set_reduce_order(order)
            digs = []
            for rep in range(3):
                Ws[:n] = to_dev(w0)
                torch.cuda.synchronize()
                dist.barrier(device_ids=[rank])
                ctx.sync_layer_ps(n, Gs, Ws, -0.01 / P)
                torch.cuda.synchronize()
                digs.append(_digest(Ws[:n]))
            res["info"][f"ps_{name}_run_to_run_identical"] = len(set(digs)) == 1
            res["digests"][f"ps_{name}"] = digs[0]
            if rank == 0:
                gs = [si.stat_dense_grad(si.rng(95, 0, q), n) for q in range(P)]
                r_ = sync.ps_update(w0, gs, -0.01 / P)
                g_ = to_host(Ws[:n])
                check(f"ps_{name}_stat_tol", err(g_, r_) <= 1e-5 and err(g_ - w0, r_ - w0) <= 1e-5)
        check("ps_rank_order_deterministic", res["info"]["ps_rank_order_run_to_run_identical"])
        if P == 2:   # AUTO at P = 2 is the peer-load kernel: rank order, deterministic too
            check("ps_auto_p2_deterministic", res["info"]["ps_auto_run_to_run_identical"])
        ctx.set_reduce_order(pos.POS_REDUCE_AUTO)

        # ---- (c) odd sizes incl. n = 16400 (shard lengths differ per rank) -------------------------
        for n_odd in (16400, 1, 130, 590080 + 77):
            Po = pos.pos_padded_size(n_odd, P)
            go = [si.exact_dense_grad(si.rng(97, n_odd % 89, q), n_odd) for q in range(P)]
            wo = si.exact_weights(si.rng(98), n_odd)
            for order in (pos.POS_REDUCE_SWITCH, pos.POS_REDUCE_RANK_ORDER, pos.POS_REDUCE_AUTO):
                ctx.set_reduce_order(order)
                Wo, Go = ctx.sym_empty(Po), ctx.sym_empty(Po)
                Wo[:n_odd] = to_dev(wo)
                Go[:n_odd] = to_dev(go[rank])
                torch.cuda.synchronize()
                ctx.sync_layer_ps(n_odd, Go, Wo, si.EXACT_ALPHA)
                torch.cuda.synchronize()
                check(f"ps_exact_{n_odd}_{order}", np.array_equal(to_host(Wo[:n_odd]), sync.ps_update(wo, go, si.EXACT_ALPHA)))
        ctx.set_reduce_order(pos.POS_REDUCE_AUTO)
        check("no_async_error", ctx.async_error() == pos.POS_OK)
        ctx.close()

        # ---- (d) watchdog: the last rank never joins a PS unit --------------------------------
        c2 = pos.Context.from_torch_distributed()
        c2.set_timeout_ms(300)
        c2.inject_fault(pos.POS_FAULT_SKIP_PS, P - 1)
        nw = 1 << 20
        Ww, Gw = c2.sym_empty(pos.pos_padded_size(nw, P)), c2.sym_empty(pos.pos_padded_size(nw, P))
        torch.cuda.synchronize()
        dist.barrier(device_ids=[rank])
        c2.sync_layer_ps(nw, Gw, Ww, 1.0)
        torch.cuda.synchronize()                        # must return (no hang)
        e = c2.async_error()
        res["info"]["watchdog_code"] = e
        if rank != P - 1:
            check("watchdog_timeout_reported", e == pos.POS_ETIMEOUT)
            check("watchdog_message", "entry barrier" in pos.lib().pos_last_error().decode())
        dist.barrier(device_ids=[rank])
        c2.close()
    except Exception:
        import traceback
        res["error"] = traceback.format_exc()
    with open(os.path.join(outdir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
    try:
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        pass


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_multi_gpu_full_model_determinism_watchdog():
    import torch.multiprocessing as mp
    world = min(_ngpu(), 8)
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, port, d), nprocs=world, join=True, start_method="spawn")
        results = [json.load(open(os.path.join(d, f"rank{r}.json"))) for r in range(world)]
    print(json.dumps([r["info"] for r in results]))
    for r in results:
        assert "error" not in r, r.get("error")
        bad = [k for k, v in r["checks"].items() if not v]
        assert not bad, (r["rank"], bad, r["info"])
    for key in results[0]["digests"]:
        assert len({r["digests"][key] for r in results}) == 1, f"replicas differ: {key}"
