"""P > 1 kernel bodies on ONE GPU (loopback): the fused PS kernel (shard reduce -> apply ->
broadcast) and the gather kernels (pack -> slot of every replica -> ready-flag
publication -> flag wait -> double-buffered reconstruction) run for P simulated ranks
with a table of local replicas instead of multicast / peer addresses (include/poseidon.h
pos_loop_*). Every replica is compared with the fp64 oracle computed from all ranks' inputs, and
the replicas with each other, bit for bit. The watchdog is exercised with an
injected fault: a rank that never packs makes the flag waits time out instead of hanging.
"""
import hashlib

import numpy as np
import pytest

import synth_inputs as si
from oracle import sync
from tests._util import err, have_gpu, to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

if have_gpu():
    import torch
    import paper_1706_03292_b200 as pos

TOL = {"bf16": 2e-3, "tf32": 2e-3, "f32": 1e-5}
_CTX = {}


def ctx(P):
    if P not in _CTX:
        _CTX[P] = pos.Context.local_sim(P)
    return _CTX[P]


def digest(t):
    return hashlib.sha256(t.detach().cpu().numpy().tobytes()).hexdigest()


# ---------------------------------------------------------------------------- PS (A6-A8) ----
PS_SIZES = [1, 10, 63, 4097, 16400, 38720, 590080, 2359808]


@pytest.mark.parametrize("P", [2, 3, 4, 8, 16])
@pytest.mark.parametrize("n", PS_SIZES)
def test_loop_ps_exact_bitwise_all_replicas(P, n):
    """Shard tails, empty shards (n < 64 P), the n = 16400 grid case of ADVICE r1; 3 iterations."""
    a = si.EXACT_ALPHA
    gs = [si.exact_dense_grad(si.rng(80, n % 97, p), n) for p in range(P)]
    w0 = si.exact_weights(si.rng(81, n % 89), n)
    Pn = pos.pos_padded_size(n, P)
    Ws, Gs = [], []
    for p in range(P):
        W = torch.full((Pn,), 7.0, device="cuda"); W[:n] = to_dev(w0)   # junk in the padding
        G = torch.zeros(Pn, device="cuda"); G[:n] = to_dev(gs[p])
        Ws.append(W); Gs.append(G)
    ref = w0
    for _ in range(3):
        ctx(P).loop_sync_layer_ps(n, Gs, Ws, a)
        ref = sync.ps_update(ref, gs, a)
    torch.cuda.synchronize()
    for p in range(P):
        assert np.array_equal(to_host(Ws[p][:n]), ref), (P, n, p)
    assert len({digest(W[:n]) for W in Ws}) == 1


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 4097, 16400, 590080])
def test_loop_ps_copy_engine_exact_and_equal_to_fused(P, n):
    """The copy-engine PS unit (POS_PS_CE: push pieces -> signal -> rank-order apply -> push shard ->
    signal -> wait) over P replicas: bitwise equal to the oracle in the exact regime over 3
    iterations, and to the fused kernel's rank-order result in the statistical regime."""
    a = si.EXACT_ALPHA
    gs = [si.exact_dense_grad(si.rng(84, n % 97, p), n) for p in range(P)]
    w0 = si.exact_weights(si.rng(85, n % 89), n)
    Pn = pos.pos_padded_size(n, P)
    Ws = [torch.zeros(Pn, device="cuda") for _ in range(P)]
    Gs = [torch.zeros(Pn, device="cuda") for _ in range(P)]
    for p in range(P):
        Ws[p][:n] = to_dev(w0)
        Gs[p][:n] = to_dev(gs[p])
    ref = w0
    for _ in range(3):
        ctx(P).loop_sync_layer_ps_ce(n, Gs, Ws, a)
        ref = sync.ps_update(ref, gs, a)
    torch.cuda.synchronize()
    assert ctx(P).async_error() == 0
    for p in range(P):
        assert np.array_equal(to_host(Ws[p][:n]), ref), (P, n, p)
    gs = [si.stat_dense_grad(si.rng(86, 0, p), n) for p in range(P)]
    w0 = si.stat_weights(si.rng(87), 1, n)[0]
    outs = []
    for fn in (ctx(P).loop_sync_layer_ps_ce, ctx(P).loop_sync_layer_ps):
        Ws = [torch.zeros(Pn, device="cuda") for _ in range(P)]
        Gs = [torch.zeros(Pn, device="cuda") for _ in range(P)]
        for p in range(P):
            Ws[p][:n] = to_dev(w0)
            Gs[p][:n] = to_dev(gs[p])
        fn(n, Gs, Ws, -0.01 / P)
        torch.cuda.synchronize()
        outs.append([digest(W[:n]) for W in Ws])
    assert len(set(outs[0])) == 1 and outs[0] == outs[1]


@pytest.mark.parametrize("P", [2, 8])
def test_loop_ps_statistical_and_repeatable(P):
    n = 2359808 + 64 * 3 + 5
    a = -0.01 / P
    gs = [si.stat_dense_grad(si.rng(82, 0, p), n) for p in range(P)]
    w0 = si.stat_weights(si.rng(83), 1, n)[0]
    Pn = pos.pos_padded_size(n, P)
    outs = []
    for rep in range(2):
        Ws = [torch.zeros(Pn, device="cuda") for _ in range(P)]
        Gs = [torch.zeros(Pn, device="cuda") for _ in range(P)]
        for p in range(P):
            Ws[p][:n] = to_dev(w0)
            Gs[p][:n] = to_dev(gs[p])
        ctx(P).loop_sync_layer_ps(n, Gs, Ws, a)
        torch.cuda.synchronize()
        outs.append([to_host(W[:n]) for W in Ws])
    ref = sync.ps_update(w0, gs, a)
    for p in range(P):
        assert err(outs[0][p], ref) <= 1e-5
        assert err(outs[0][p] - w0, ref - w0) <= 1e-5       # fp32 end to end
        assert np.array_equal(outs[0][p], outs[0][0])        # replicas identical
        assert np.array_equal(outs[1][p], outs[0][p])        # fixed rank order: run to run


# --------------------------------------------------------------------------- SFB (A2-A4b) ----
def loop_fc_run(P, K, M, N, dtype, in_dtype, regime, iters=3, seed=0, bias=True):
    Us, Vs = [], []
    for p in range(P):
        g = si.rng(seed, 3, p)
        if regime == "exact":
            u, v = si.exact_factors(g, K, M, N)
        else:
            u, v = si.stat_factors(g, K, M, N, "bf16" if dtype == "bf16" else "f32")
        Us.append(u); Vs.append(v)
    g = si.rng(seed, 4)
    if regime == "exact":
        W0, b0 = si.exact_weights(g, M, N), si.exact_weights(g, M)
        a = si.EXACT_ALPHA
    else:
        W0, b0 = si.stat_weights(g, M, N), si.stat_weights(g, 1, M)[0]
        a = -0.01 / P
    Wd = [to_dev(W0) for _ in range(P)]
    bd = [to_dev(b0) for _ in range(P)] if bias else None
    lf = pos.LoopFC(ctx(P), M, N, K, Wd, bd, dtype)
    st = "bf16" if in_dtype == "bf16" else "f32"
    us = [to_dev(u, st) for u in Us]
    vs = [to_dev(v, st) for v in Vs]
    Wr, br = W0, (b0 if bias else None)
    for _ in range(iters):
        lf.sync(us, vs, a)
        Wr, br = sync.sfb_update(Wr, br, Us, Vs, a)
    torch.cuda.synchronize()
    lf.close()
    return W0, Wd, bd, Wr, br


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype,in_dtype", [("bf16", "bf16"), ("tf32", "f32"), ("f32", "f32")])
@pytest.mark.parametrize("MN", [(64, 64), (65, 132), (1000, 4100), (257, 1028)])
def test_loop_fc_exact_bitwise_3iter(P, dtype, in_dtype, MN):
    """bf16 / tf32: flag-mode gather (double buffer selected on the device, 3 iterations alternate
    buffers); f32: barrier-mode layout + SIMT reconstruction."""
    M, N = MN
    K = 8 if P < 8 else 4
    _, Wd, bd, Wr, br = loop_fc_run(P, K, M, N, dtype, in_dtype, "exact")
    for p in range(P):
        assert np.array_equal(to_host(Wd[p]), Wr), (P, dtype, MN, p)
        assert np.array_equal(to_host(bd[p]), br), (P, dtype, MN, p)


def test_loop_fc_ragged_n_uses_barrier_layout():
    """N % 4 != 0: no tensor-core plan, so the barrier-mode (single buffer) gather + SIMT path."""
    for dtype in ("bf16", "tf32"):
        _, Wd, bd, Wr, br = loop_fc_run(4, 8, 33, 131, dtype, "f32", "exact", iters=2)
        for p in range(4):
            assert np.array_equal(to_host(Wd[p]), Wr)
            assert np.array_equal(to_host(bd[p]), br)


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_loop_fc_statistical(dtype):
    P = 4
    W0, Wd, bd, Wr, br = loop_fc_run(P, 32, 1000, 4096, dtype, "bf16" if dtype == "bf16" else "f32",
                                     "stat", iters=2)
    for p in range(P):
        g = to_host(Wd[p])
        assert err(g, Wr) <= TOL[dtype] and err(g - W0, Wr - W0) <= TOL[dtype]
        assert err(to_host(bd[p]), br) <= TOL[dtype]
    assert len({digest(W) for W in Wd}) == 1


def test_loop_fc_alexnet_fc6_kp1024_full_compare():
    """C1 AlexNet fc6 (4096 x 9216) at K = 128, P = 8 (K*P = 1024: the CTA-pair kernel, as in the
    bench at 8 GPUs): every element of every replica, exact regime bitwise (2 iterations)."""
    P, K, M, N = 8, 128, 4096, 9216
    _, Wd, bd, Wr, br = loop_fc_run(P, K, M, N, "bf16", "bf16", "exact", iters=2, seed=5)
    for p in range(P):
        assert np.array_equal(to_host(Wd[p]), Wr), p
        assert np.array_equal(to_host(bd[p]), br), p


def test_loop_fc_alexnet_fc6_kp1024_statistical_full():
    P, K, M, N = 8, 128, 4096, 9216
    W0, Wd, bd, Wr, br = loop_fc_run(P, K, M, N, "bf16", "bf16", "stat", iters=1, seed=6, bias=False)
    g = to_host(Wd[0])
    assert err(g, Wr) <= TOL["bf16"] and err(g - W0, Wr - W0) <= TOL["bf16"]
    assert len({digest(W) for W in Wd}) == 1


# ------------------------------------------------------------------------------ watchdog ----
def test_watchdog_flag_wait_times_out_instead_of_hanging():
    """Rank 1 never packs (injected fault): every replica's ready-flag wait gives up after the
    context's timeout and the context reports POS_ETIMEOUT (sticky) instead of hanging."""
    c = pos.Context.local_sim(2)
    c.set_timeout_ms(100)
    c.inject_fault(pos.POS_FAULT_SKIP_PACK, 1)
    M, N, K = 256, 256, 8
    Wd = [torch.zeros(M, N, device="cuda") for _ in range(2)]
    lf = pos.LoopFC(c, M, N, K, Wd, None, "bf16")
    u = torch.ones(K, M, device="cuda", dtype=torch.bfloat16)
    v = torch.ones(K, N, device="cuda", dtype=torch.bfloat16)
    lf.sync([u, u], [v, v], -1.0)
    torch.cuda.synchronize()                       # returns: the kernels did not hang
    assert c.async_error() == pos.POS_ETIMEOUT
    assert "flags" in pos.lib().pos_last_error().decode()
    with pytest.raises(pos.PoseidonError) as e:    # sticky
        lf.sync([u, u], [v, v], -1.0)
    assert e.value.code == pos.POS_ETIMEOUT
    lf.close()
    c.close()
    # a fresh context is unaffected
    c2 = pos.Context.local_sim(2)
    assert c2.async_error() == pos.POS_OK
    c2.close()
