"""Real multi-GPU synchronisation over NCCL (T7/T8 of SURVEY §8(c)): one process per GPU, every
rank's result compared with the fp64 oracle computed from ALL ranks' inputs, and replicas compared
with each other bit for bit.

Runs with as many GPUs as are visible (>= 2); skipped otherwise.
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

    import paper_1706_03292_b200 as pos
    import synth_inputs as si
    from oracle import sync
    from tests._util import err, to_dev, to_host

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    res = {"rank": rank, "checks": {}, "digests": {}}
    P = world

    def check(name, ok):
        res["checks"][name] = bool(ok)

    try:
        ctx = pos.Context.from_torch_distributed()
        a = si.EXACT_ALPHA
        # ---- (a) SFB one-shot, exact regime, FC 4096 x 4096, K = 32 --------------------------
        M, N, K = 4096, 4096, 32
        Us, Vs = zip(*(si.exact_factors(si.rng(40, 0, p), K, M, N) for p in range(P)))
        W0 = si.exact_weights(si.rng(40, 1), M, N)
        b0 = si.exact_weights(si.rng(40, 2), M)
        W, b = to_dev(W0), to_dev(b0)
        ctx.sync_layer_sfb(to_dev(Us[rank], "bf16"), to_dev(Vs[rank], "bf16"), W, b, a, "bf16")
        torch.cuda.synchronize()
        Wr, br = sync.sfb_update(W0, b0, Us, Vs, a)
        check("sfb_exact_W", np.array_equal(to_host(W), Wr))
        check("sfb_exact_b", np.array_equal(to_host(b), br))
        res["digests"]["sfb"] = _digest(W) + _digest(b)
        # ---- (b) PS one-shot, dense 2,359,808 (VGG conv 512x512x3x3 + bias) -------------------
        n = 2359808
        gs = [si.exact_dense_grad(si.rng(41, 0, p), n) for p in range(P)]
        w0 = si.exact_weights(si.rng(41, 1), n)
        Pn = pos.pos_padded_size(n, P)
        Wd = torch.zeros(Pn, device=dev); Wd[:n] = to_dev(w0)
        Gd = torch.full((Pn,), 3.0, device=dev); Gd[:n] = to_dev(gs[rank])
        ctx.sync_layer_ps(n, Gd, Wd, a)
        torch.cuda.synchronize()
        check("ps_exact", np.array_equal(to_host(Wd[:n]), sync.ps_update(w0, gs, a)))
        res["digests"]["ps"] = _digest(Wd[:n])
        # ---- (b2) PS through the fused NVLS kernel (grad and W in symmetric memory) -------------
        Ws = ctx.sym_empty(Pn)
        Gs = ctx.sym_empty(Pn)
        check("symm_alloc", ctx.is_symmetric(Ws) and ctx.is_symmetric(Gs) and not ctx.is_symmetric(Wd))
        Ws[:n] = to_dev(w0)
        Gs[:n] = to_dev(gs[rank])
        torch.cuda.synchronize()
        ctx.sync_layer_ps(n, Gs, Ws, a)
        torch.cuda.synchronize()
        check("ps_nvls_exact", np.array_equal(to_host(Ws[:n]), sync.ps_update(w0, gs, a)))
        res["digests"]["ps_nvls"] = _digest(Ws[:n])
        # odd sizes: shard tails, tiny layers with empty shards
        for n_odd in (1, 10, 4097, 1792 + 36928):
            P_o = pos.pos_padded_size(n_odd, P)
            go = [si.exact_dense_grad(si.rng(48, n_odd % 97, p), n_odd) for p in range(P)]
            wo = si.exact_weights(si.rng(48, 1), n_odd)
            Wo, Go = ctx.sym_empty(P_o), ctx.sym_empty(P_o)
            Wo[:n_odd] = to_dev(wo)
            Go[:n_odd] = to_dev(go[rank])
            torch.cuda.synchronize()
            ctx.sync_layer_ps(n_odd, Go, Wo, a)
            torch.cuda.synchronize()
            check(f"ps_nvls_exact_{n_odd}", np.array_equal(to_host(Wo[:n_odd]), sync.ps_update(wo, go, a)))
        # ---- (c) FC forced onto the PS path == SFB result ------------------------------------
        M2, N2, K2 = 1000, 4100, 8
        Us2, Vs2 = zip(*(si.exact_factors(si.rng(42, 0, p), K2, M2, N2) for p in range(P)))
        W20 = si.exact_weights(si.rng(42, 1), M2, N2)
        b20 = si.exact_weights(si.rng(42, 2), M2)
        nn_ = M2 * N2 + M2
        Pn2 = pos.pos_padded_size(nn_, P)
        flat = torch.zeros(Pn2, device=dev)
        flat[:M2 * N2] = to_dev(W20).reshape(-1)
        flat[M2 * N2:nn_] = to_dev(b20)
        grad = torch.empty(Pn2, device=dev)
        ctx.sync_layer_fc_ps(to_dev(Us2[rank], "bf16"), to_dev(Vs2[rank], "bf16"), grad, flat, True, a, "bf16")
        torch.cuda.synchronize()
        Wr2, br2 = sync.sfb_update(W20, b20, Us2, Vs2, a)
        check("fc_ps_W", np.array_equal(to_host(flat[:M2 * N2]).reshape(M2, N2), Wr2))
        check("fc_ps_b", np.array_equal(to_host(flat[M2 * N2:nn_]), br2))
        res["digests"]["fc_ps"] = _digest(flat[:nn_])
        # ---- (d) statistical regime SFB, tolerance + replica identity --------------------------
        Us3, Vs3 = zip(*(si.stat_factors(si.rng(43, 0, p), K, M, N, "bf16") for p in range(P)))
        W30 = si.stat_weights(si.rng(43, 1), M, N)
        W3 = to_dev(W30)
        ctx.sync_layer_sfb(to_dev(Us3[rank], "bf16"), to_dev(Vs3[rank], "bf16"), W3, None, -0.01 / P, "bf16")
        torch.cuda.synchronize()
        Wr3, _ = sync.sfb_update(W30, None, Us3, Vs3, -0.01 / P)
        g3 = to_host(W3)
        check("sfb_stat_W", err(g3, Wr3) <= 2e-3)
        check("sfb_stat_dW", err(g3 - W30, Wr3 - W30) <= 2e-3)
        res["digests"]["sfb_stat"] = _digest(W3)
        # ---- (f) scheduler SFB: tf32 (flag-mode gather, double buffer), fp32 (barrier-mode
        #          multicast + SIMT reconstruction) and a K*P = 1024 layer (single-CTA kernel by default,
        #          then the CTA-pair kernel forced); 3 iterations
        def run_dtype(dt, in_dt, Kx, Mx, Nx, iters=3):
            sch = pos.Scheduler(ctx, 1)
            U, V = zip(*(si.exact_factors(si.rng(49, Kx, p), Kx, Mx, Nx) for p in range(P)))
            w0_ = si.exact_weights(si.rng(49, 1), Mx, Nx)
            b0_ = si.exact_weights(si.rng(49, 2), Mx)
            Wx, Bx = to_dev(w0_), to_dev(b0_)
            assert sch.add_fc(0, Mx, Nx, Kx, Wx, Bx, None, dt, in_dt) == pos.POS_SCHEME_SFB
            st = "bf16" if in_dt == pos.POS_IN_BF16 else "f32"
            u, v = to_dev(U[rank], st), to_dev(V[rank], st)
            for _ in range(iters):
                sch.begin(a)
                sch.factors_ready(0, u, v, torch.cuda.current_stream())
                sch.end(torch.cuda.current_stream())
            torch.cuda.synchronize()
            wr, br_ = w0_, b0_
            for _ in range(iters):
                wr, br_ = sync.sfb_update(wr, br_, U, V, a)
            ok = np.array_equal(to_host(Wx), wr) and np.array_equal(to_host(Bx), br_)
            sch.close()
            return ok
        check("sched_tf32_flags_3iter", run_dtype("tf32", pos.POS_IN_F32, 16, 1000, 1028))
        check("sched_f32_barrier_3iter", run_dtype("f32", pos.POS_IN_F32, 16, 300, 132))
        check("sched_kp1024_3iter", run_dtype("bf16", pos.POS_IN_BF16, 1024 // P, 2000, 4100))
        # the CTA-pair (cluster) kernel is off at P > 1 by default; forced on, eager, it still works
        os.environ["POS_SFB_PAIR"] = "1"
        try:
            check("sched_pair_forced_3iter", run_dtype("bf16", pos.POS_IN_BF16, 1024 // P, 2000, 4100))
        finally:
            del os.environ["POS_SFB_PAIR"]
        # ---- (e) WFBP scheduler: FC (SFB) + bucket + dense; WFBP == sequential, both == oracle --
        def run_sched(sequential, graph, symm_dense=False, iters=1):
            alloc = (lambda k: ctx.sym_empty(k)) if symm_dense else (lambda k: torch.zeros(k, device=dev))
            sch = pos.Scheduler(ctx, 5, timing="apply", sequential=sequential)
            sizes = [1792, 36928]
            nb = sum(sizes)
            Pb = pos.pos_padded_size(nb, P)
            wb0 = si.exact_weights(si.rng(44, 0), nb)
            gb = [si.exact_dense_grad(si.rng(44, 1, p), nb) for p in range(P)]
            Wb = alloc(Pb); Wb[:nb] = to_dev(wb0)
            Gb = alloc(Pb)
            sch.add_dense_bucket(0, sizes, Wb, Gb)
            n2 = 590080
            Pd = pos.pos_padded_size(n2, P)
            wd0 = si.exact_weights(si.rng(45, 0), n2)
            gd = [si.exact_dense_grad(si.rng(45, 1, p), n2) for p in range(P)]
            Wq = alloc(Pd); Wq[:n2] = to_dev(wd0)
            Gq = alloc(Pd)
            sch.add_dense(2, n2, Wq, Gq)
            Mf, Nf, Kf = 4096, 9216, 16
            Uf, Vf = zip(*(si.exact_factors(si.rng(46, 0, p), Kf, Mf, Nf) for p in range(P)))
            wf0 = si.exact_weights(si.rng(46, 1), Mf, Nf)
            bf0 = si.exact_weights(si.rng(46, 2), Mf)
            Wf, Bf = to_dev(wf0), to_dev(bf0)
            assert sch.add_fc(3, Mf, Nf, Kf, Wf, Bf, None, "bf16", pos.POS_IN_BF16) == pos.POS_SCHEME_SFB
            Mg, Ng, Kg = 1000, 4096, 16
            Ug, Vg = zip(*(si.exact_factors(si.rng(47, 0, p), Kg, Mg, Ng) for p in range(P)))
            wg0 = si.exact_weights(si.rng(47, 1), Mg, Ng)
            Wg = to_dev(wg0)
            sch.add_fc(4, Mg, Ng, Kg, Wg, None, None, "bf16", pos.POS_IN_BF16)
            uf, vf = to_dev(Uf[rank], "bf16"), to_dev(Vf[rank], "bf16")
            ug, vg = to_dev(Ug[rank], "bf16"), to_dev(Vg[rank], "bf16")

            def fill():
                Gb[:nb] = to_dev(gb[rank]); Gq[:n2] = to_dev(gd[rank])

            def step(stream):
                sch.begin(a)
                sch.factors_ready(4, ug, vg, stream)
                sch.factors_ready(3, uf, vf, stream)
                sch.grad_ready(2, stream)
                sch.grad_ready(1, stream)
                sch.grad_ready(0, stream)
                sch.end(stream)

            fill()
            torch.cuda.synchronize()
            if graph:   # one captured iteration, replayed: device-side state must advance per replay
                gr = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.graph(gr, stream=cs, capture_error_mode="thread_local"):
                    step(torch.cuda.current_stream())
                torch.cuda.synchronize()
                for it in range(iters):
                    if it:
                        fill()   # the NCCL path reduces in place
                    gr.replay()
            else:
                for it in range(iters):
                    if it:
                        fill()
                    step(torch.cuda.current_stream())
            torch.cuda.synchronize()
            wb1, wd1, wf1, bf1, wg1 = wb0, wd0, wf0, bf0, wg0
            for _ in range(iters):
                wb1 = sync.ps_update(wb1, gb, a)
                wd1 = sync.ps_update(wd1, gd, a)
                wf1, bf1 = sync.sfb_update(wf1, bf1, Uf, Vf, a)
                wg1, _ = sync.sfb_update(wg1, None, Ug, Vg, a)
            ok = np.array_equal(to_host(Wb[:nb]), wb1)
            ok &= np.array_equal(to_host(Wq[:n2]), wd1)
            ok &= np.array_equal(to_host(Wf), wf1) and np.array_equal(to_host(Bf), bf1)
            ok &= np.array_equal(to_host(Wg), wg1)
            dig = _digest(Wb[:nb]) + _digest(Wq[:n2]) + _digest(Wf) + _digest(Wg)
            sch.close()
            return bool(ok), dig

        ok_w, dig_w = run_sched(False, False)
        ok_s, dig_s = run_sched(True, False)
        ok_g, dig_g = run_sched(False, True)
        ok_n, dig_n = run_sched(False, True, symm_dense=True)
        ok_ns, dig_ns = run_sched(True, False, symm_dense=True)
        # several iterations: the double-buffered flag-mode gather alternates buffers (by a device
        # counter, so a single replayed graph alternates too) and the flags keep advancing
        ok_n5, dig_n5 = run_sched(False, True, symm_dense=True, iters=5)
        ok_w5, dig_w5 = run_sched(False, False, symm_dense=True, iters=5)
        ok_s5, dig_s5 = run_sched(True, False, iters=5)
        check("sched_nvls_graph_5iter_oracle", ok_n5)
        check("sched_nvls_eager_5iter_oracle", ok_w5)
        check("sched_seq_5iter_oracle", ok_s5)
        check("sched_5iter_replicas_agree", dig_n5 == dig_w5 == dig_s5)
        check("sched_nvls_graph_oracle", ok_n)
        check("sched_nvls_seq_oracle", ok_ns)
        check("sched_wfbp_oracle", ok_w)
        check("sched_seq_oracle", ok_s)
        check("sched_graph_oracle", ok_g)
        check("sched_wfbp_eq_seq", dig_w == dig_s == dig_g)
        check("sched_nvls_eq_nccl", dig_n == dig_ns == dig_w)
        res["digests"]["sched"] = dig_w
        ctx.close()
    except Exception as e:  # report, do not hang the other ranks silently
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
def test_multi_gpu_nccl_parity_and_replicas():
    import torch.multiprocessing as mp
    world = min(_ngpu(), 8)
    port = _free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, port, d), nprocs=world, join=True, start_method="spawn")
        results = [json.load(open(os.path.join(d, f"rank{r}.json"))) for r in range(world)]
    for r in results:
        assert "error" not in r, r.get("error")
        bad = [k for k, v in r["checks"].items() if not v]
        assert not bad, (r["rank"], bad)
    for key in results[0]["digests"]:
        assert len({r["digests"][key] for r in results}) == 1, f"replicas differ: {key}"
