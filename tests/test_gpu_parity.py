"""GPU parity: CUDA path (through the C ABI) vs the fp64 oracle on identical seeded inputs.

Regimes:
  exact       integer factors / grads, W = j/256, alpha = -2^-12: every product and partial sum is
              exact in fp32, so the GPU result must equal the oracle BITWISE for every dtype, scheme,
              P and tile edge (a mismatch is an indexing/tiling bug).
  statistical u = 2^-5 N(0,1), v = ReLU(N(0,1)) rounded to the device dtype, W ~ U(+-1/sqrt N):
              err(W') and err(dW) <= 2e-3 for bf16/tf32, <= 1e-5 for f32 (north_star; reading S15).
"""
import os

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


def factors(seed, P, K, M, N, regime, dtype):
    Us, Vs = [], []
    for p in range(P):
        g = si.rng(seed, 1, p)
        if regime == "exact":
            u, v = si.exact_factors(g, K, M, N)
        else:
            u, v = si.stat_factors(g, K, M, N, "bf16" if dtype == "bf16" else "f32")
        Us.append(u)
        Vs.append(v)
    return Us, Vs


def run_sfb(P, K, M, N, dtype, in_dtype, regime, seed=0, alpha=None, zero_w=False, bias=True):
    Us, Vs = factors(seed, P, K, M, N, regime, dtype)
    g = si.rng(seed, 2)
    if zero_w:
        W = np.zeros((M, N), np.float32)
        b = np.zeros(M, np.float32)
    elif regime == "exact":
        W, b = si.exact_weights(g, M, N), si.exact_weights(g, M)
    else:
        W, b = si.stat_weights(g, M, N), si.stat_weights(g, 1, M)[0]
    if alpha is None:
        alpha = si.EXACT_ALPHA if regime == "exact" else -0.01 / P
    st = "bf16" if in_dtype == "bf16" else "f32"
    us = [to_dev(u, st) for u in Us]
    vs = [to_dev(v, st) for v in Vs]
    Wd, bd = to_dev(W), to_dev(b) if bias else None
    ctx(P).sim_sync_layer_sfb(us, vs, Wd, bd, alpha, dtype)
    torch.cuda.synchronize()
    W_ref, b_ref = sync.sfb_update(W, b if bias else None, Us, Vs, alpha)
    return W, b, to_host(Wd), to_host(bd) if bias else None, W_ref, b_ref


# ----------------------------------------------------------------------------- C0, exact ----
@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32"])
@pytest.mark.parametrize("in_dtype", ["bf16", "f32"])
@pytest.mark.parametrize("P", [1, 2])
def test_c0_sfb_exact_bitwise(P, dtype, in_dtype):
    _, _, Wg, bg, Wr, br = run_sfb(P, 8, 64, 64, dtype, in_dtype, "exact")
    assert np.array_equal(Wg, Wr)
    assert np.array_equal(bg, br)


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32"])
@pytest.mark.parametrize("P", [1, 2])
def test_c0_sfb_equals_ps_exact_bitwise(P, dtype):
    """SFB and PS give identical W: the PS path's per-worker FC gradient is formed on
    the GPU by the reconstruction kernel in overwrite mode, then reduced and applied."""
    K, M, N = 8, 64, 64
    Us, Vs = factors(3, P, K, M, N, "exact", dtype)
    W = si.exact_weights(si.rng(3, 2), M, N)
    a = si.EXACT_ALPHA
    st = "bf16" if dtype == "bf16" else "f32"
    # SFB
    W_sfb = to_dev(W)
    ctx(P).sim_sync_layer_sfb([to_dev(u, st) for u in Us], [to_dev(v, st) for v in Vs], W_sfb, None, a, dtype)
    # PS: per-worker dense gradient via the GPU kernels (pack + reconstruct, overwrite, alpha = 1)
    grads = []
    R = pos.pos_factor_row_elems(M, N)
    for u, v in zip(Us, Vs):
        rows = pos.pos_factor_slot_rows(K, pos.DTYPES[dtype])
        slot = torch.empty(rows * R, dtype=torch.bfloat16 if dtype == "bf16" else torch.float32, device="cuda")
        pos.pos_pack_factors(to_dev(u, st), to_dev(v, st), slot, pos.DTYPES[dtype])
        gd = torch.empty(M * N, dtype=torch.float32, device="cuda")
        pos.pos_reconstruct_apply(M, N, K, pos.DTYPES[dtype], slot, gd, None, 1.0, accumulate=False)
        grads.append(gd)
    W_ps = to_dev(W).reshape(-1)
    ctx(P).sim_sync_layer_ps(grads, W_ps, a)
    torch.cuda.synchronize()
    W_ref, _ = sync.sfb_update(W, None, Us, Vs, a)
    assert np.array_equal(to_host(W_sfb), W_ref)
    assert np.array_equal(to_host(W_ps).reshape(M, N), W_ref)
    for gd, u, v in zip(grads, Us, Vs):
        assert np.array_equal(to_host(gd).reshape(M, N), sync.fc_grad(u, v))


# ------------------------------------------------------------------------ C0, statistical ----
@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32"])
@pytest.mark.parametrize("P", [1, 2])
@pytest.mark.parametrize("seed", range(10))
def test_c0_sfb_statistical(P, dtype, seed):
    W, _, Wg, bg, Wr, br = run_sfb(P, 8, 64, 64, dtype, "bf16" if dtype == "bf16" else "f32", "stat", seed)
    assert err(Wg, Wr) <= TOL[dtype]
    assert err(Wg - W, Wr - W) <= TOL[dtype]
    assert err(bg, br) <= TOL[dtype]
    # W = 0, alpha = -1: W' = dW exactly exposes the reconstruction error
    _, _, Wg, bg, Wr, br = run_sfb(P, 8, 64, 64, dtype, "bf16" if dtype == "bf16" else "f32", "stat", seed,
                                   alpha=-1.0, zero_w=True)
    assert err(Wg, Wr) <= TOL[dtype]
    assert err(bg, br) <= TOL[dtype]


# ------------------------------------------------------------------------- tile edges (T6) ----
EDGE = [1, 7, 63, 64, 65, 127, 129, 1000, 4097]
TC_N = [4, 36, 260, 1028, 4100]   # N % 4 == 0: tensor-core path with ragged n tiles


@pytest.mark.parametrize("M", EDGE)
@pytest.mark.parametrize("N", EDGE + TC_N)
def test_tile_edges_exact_bitwise_bf16(M, N):
    _, _, Wg, bg, Wr, br = run_sfb(2, 8, M, N, "bf16", "bf16", "exact", seed=M * 7 + N)
    assert np.array_equal(Wg, Wr), (M, N)
    assert np.array_equal(bg, br)


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32"])
@pytest.mark.parametrize("K", [1, 8, 32])
@pytest.mark.parametrize("P", [1, 2])
@pytest.mark.parametrize("MN", [(1, 4), (65, 129), (129, 260), (1000, 4100), (4097, 64)])
def test_tile_edges_exact_bitwise_k_p(MN, K, P, dtype):
    M, N = MN
    _, _, Wg, bg, Wr, br = run_sfb(P, K, M, N, dtype, "f32", "exact", seed=K + 10 * P)
    assert np.array_equal(Wg, Wr)
    assert np.array_equal(bg, br)


# ------------------------------------------------------- CTA-pair kernel (cta_group::2) ----
# The pair kernel (256-row tiles, each CTA holding half of the V columns) is chosen for
# K*P >= 1024 (sfb_tc.cu POS_SFB_PAIR_KP); POS_SFB_PAIR=1 / 0 forces it on / off at plan time so that
# both kernels are checked on the same ragged shapes.
PAIR_MN = [(1, 4), (65, 129), (129, 260), (255, 132), (257, 1028), (1000, 4100), (4097, 64)]


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
@pytest.mark.parametrize("KP", [(1, 1), (8, 2), (32, 8), (40, 7)])
@pytest.mark.parametrize("MN", PAIR_MN)
def test_pair_kernel_exact_bitwise(MN, KP, dtype, monkeypatch):
    monkeypatch.setenv("POS_SFB_PAIR", "1")
    (M, N), (K, P) = MN, KP
    _, _, Wg, bg, Wr, br = run_sfb(P, K, M, N, dtype, "f32", "exact", seed=M + N + K)
    assert np.array_equal(Wg, Wr), (M, N, K, P)
    assert np.array_equal(bg, br)


@pytest.mark.parametrize("pair", ["0", "1"])
@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_pair_and_single_kernels_statistical_large_kp(pair, dtype, monkeypatch):
    """K*P = 512 (AlexNet-like fc7 at P = 4): both kernels within the north_star tolerance."""
    monkeypatch.setenv("POS_SFB_PAIR", pair)
    W, _, Wg, bg, Wr, br = run_sfb(4, 128, 1000, 1028, dtype, "bf16" if dtype == "bf16" else "f32",
                                   "stat", seed=5)
    assert err(Wg, Wr) <= TOL[dtype]
    assert err(Wg - W, Wr - W) <= TOL[dtype]
    assert err(bg, br) <= TOL[dtype]


# ---------------------------------------------------------------------- full-size layers ----
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("layer", [(4096, 25088, 32, 1), (21841, 4096, 32, 1), (4096, 4096, 32, 8),
                                   (1000, 4096, 32, 2)])
def test_full_size_layers_exact_bitwise(layer, dtype):
    """Bench shapes (C3 VGG19-22K fc6/fc8 at P = 1; fc7 at K*P = 256), launched exactly as the bench
    launches them (tensor-core kernel, one CTA per SM), compared element by element. f32: the 3xTF32
    rows (3 K P of them) through the same kernel."""
    M, N, K, P = layer
    _, _, Wg, bg, Wr, br = run_sfb(P, K, M, N, dtype, "bf16" if dtype == "bf16" else "f32", "exact", seed=11)
    assert np.array_equal(Wg, Wr)
    assert np.array_equal(bg, br)


@pytest.mark.parametrize("layer", [(4096, 25088, 32, 1), (21841, 4096, 32, 2)])
def test_full_size_f32_statistical(layer):
    """fp32 factors (3xTF32, reading S16) at the bench's largest shapes, statistical regime: every
    element of W' and dW within the fp32 tolerance of the fp64 oracle."""
    M, N, K, P = layer
    W, b, Wg, bg, Wr, br = run_sfb(P, K, M, N, "f32", "f32", "stat", seed=12)
    assert err(Wg, Wr) <= TOL["f32"]
    assert err(Wg - W, Wr - W) <= TOL["f32"]
    assert err(bg - b, br - b) <= TOL["f32"]


def test_alexnet_kp1024_full():
    """C1 AlexNet fc6 4096 x 9216 at K = 128, P = 8 (K*P = 1024, the CTA-pair kernel): statistical
    regime, EVERY element compared with the fp64 oracle (W' and dW), and the exact regime bitwise."""
    M, N, K, P = 4096, 9216, 128, 8
    W, _, Wg, _, Wr, _ = run_sfb(P, K, M, N, "bf16", "bf16", "stat", seed=21, bias=False)
    assert err(Wg, Wr) <= TOL["bf16"]
    assert err(Wg - W, Wr - W) <= TOL["bf16"]
    _, _, Wg, bg, Wr, br = run_sfb(P, K, M, N, "bf16", "bf16", "exact", seed=22)
    assert np.array_equal(Wg, Wr) and np.array_equal(bg, br)


# ------------------------------------------------------------------------ degenerate cases ----
def test_alpha_zero_and_zero_factors_leave_w_unchanged():
    M, N, K = 129, 260, 8
    for dtype in ("bf16", "tf32", "f32"):
        W, b, Wg, bg, _, _ = run_sfb(2, K, M, N, dtype, "f32", "stat", alpha=0.0)
        assert np.array_equal(Wg, W.astype(np.float64)) and np.array_equal(bg, b.astype(np.float64))
    W = si.stat_weights(si.rng(5), M, N)
    Wd = to_dev(W)
    z = torch.zeros(K, M, device="cuda")
    v = to_dev(si.stat_factors(si.rng(6), K, M, N, "f32")[1])
    ctx(2).sim_sync_layer_sfb([z, z], [v, v], Wd, None, -1.0, "bf16")
    torch.cuda.synchronize()
    assert np.array_equal(to_host(Wd), W.astype(np.float64))


def test_deterministic_repeat():
    M, N, K = 1000, 4100, 32
    Us, Vs = factors(8, 2, K, M, N, "stat", "bf16")
    W = si.stat_weights(si.rng(8), M, N)
    outs = []
    for _ in range(2):
        Wd = to_dev(W)
        ctx(2).sim_sync_layer_sfb([to_dev(u, "bf16") for u in Us], [to_dev(v, "bf16") for v in Vs], Wd,
                                  None, -0.01, "bf16")
        torch.cuda.synchronize()
        outs.append(Wd.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


# ------------------------------------------------------------------------------ PS kernels ----
@pytest.mark.parametrize("n", [1, 3, 4, 5, 63, 64, 65, 1000, 4097, 2359808])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_ps_sim_exact_bitwise(n, P):
    grads = [si.exact_dense_grad(si.rng(9, n % 101, p), n) for p in range(P)]
    W = si.exact_weights(si.rng(9, 1), n)
    Wd = to_dev(W)
    ctx(P).sim_sync_layer_ps([to_dev(g) for g in grads], Wd, si.EXACT_ALPHA)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(Wd), sync.ps_update(W, grads, si.EXACT_ALPHA))


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
@pytest.mark.parametrize("count", [1, 5, 64, 1001, 1 << 20])
def test_ps_apply_alignment_and_tails(offset, count):
    g = si.stat_dense_grad(si.rng(10), count + 8)
    W = si.stat_weights(si.rng(11), 1, count + 8)[0]
    gd, Wd = to_dev(g), to_dev(W)
    pos.pos_ps_apply(gd[offset:], Wd[offset:], count, -0.5)
    torch.cuda.synchronize()
    ref = W.astype(np.float64).copy()
    ref[offset:offset + count] += -0.5 * g[offset:offset + count].astype(np.float64)
    got = to_host(Wd)
    assert np.array_equal(got[:offset], ref[:offset]) and np.array_equal(got[offset + count:], ref[offset + count:])
    assert err(got, ref) <= 1e-7


def test_dense_ps_one_gpu_world1():
    """pos_sync_layer_ps on a world-1 context: local apply over [0, n), tail of grad zeroed."""
    c = pos.Context.from_unique_id(bytes(128), 1, 0)
    n = 2359808
    Ppad = pos.pos_padded_size(n, 1)
    g = si.exact_dense_grad(si.rng(12), n)
    W = si.exact_weights(si.rng(13), n)
    gd = torch.full((Ppad,), 7.0, device="cuda")
    gd[:n] = to_dev(g)
    Wd = torch.zeros(Ppad, device="cuda")
    Wd[:n] = to_dev(W)
    c.sync_layer_ps(n, gd, Wd, si.EXACT_ALPHA)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(Wd[:n]), sync.ps_update(W, [g], si.EXACT_ALPHA))
    assert torch.count_nonzero(gd[n:]).item() == 0
    c.close()


# -------------------------------------------------------------------------------- pack A2 ----
def _tf32_rna(x):
    """fp32 -> tf32 (10 explicit mantissa bits), round to nearest with ties away from zero: add half
    a tf32 ulp to the magnitude bits and truncate (IEEE sign-magnitude; finite inputs)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((b + 0x1000) & 0xFFFFE000).astype(np.uint32)).view(np.float32)


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32"])
def test_pack_layout(dtype):
    K, M, N = 5, 13, 7
    g = si.rng(14)
    u = g.standard_normal((K, M)).astype(np.float32)
    v = g.standard_normal((K, N)).astype(np.float32)
    R = pos.pos_factor_row_elems(M, N)
    assert R == 64 + 64
    rows = pos.pos_factor_slot_rows(K, pos.DTYPES[dtype])
    ffma = os.environ.get("POS_F32_FFMA") == "1"      # exact-fp32 mode: one plain row per pair
    assert rows == (3 * K if dtype == "f32" and not ffma else K)
    ud, vd = to_dev(u), to_dev(v)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    slot = torch.full((rows, R), 99.0, dtype=tdt, device="cuda")
    pos.pos_pack_factors(ud, vd, slot, pos.DTYPES[dtype])
    torch.cuda.synchronize()
    exp = torch.zeros(rows, R, dtype=tdt)
    if dtype != "f32" or ffma:
        exp[:, :M] = torch.from_numpy(u).to(tdt)          # torch's CPU RNE cast (bf16); fp32 copy
        exp[:, 64:64 + N] = torch.from_numpy(v).to(tdt)
        exp[:, 64 + N] = 1.0                              # ones column (fused bias gradient)
    else:
        # 3xTF32 blocks (reading S16): (hi u, hi v), (hi u, lo v), (lo u, hi v)
        hi = {"u": _tf32_rna(u), "v": _tf32_rna(v)}
        lo = {"u": _tf32_rna(u - hi["u"]), "v": _tf32_rna(v - hi["v"])}
        assert np.all(np.abs(hi["u"] + lo["u"] - u) <= 2.0 ** -21 * np.abs(u))
        for blk, (pu, pv, one) in enumerate([(hi, hi, 1.0), (hi, lo, 0.0), (lo, hi, 1.0)]):
            r = slice(blk * K, (blk + 1) * K)
            exp[r, :M] = torch.from_numpy(pu["u"])
            exp[r, 64:64 + N] = torch.from_numpy(pv["v"])
            exp[r, 64 + N] = one
    assert torch.equal(slot.cpu(), exp)
