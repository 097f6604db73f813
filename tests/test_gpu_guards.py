"""Out-of-bounds write detection without compute-sanitizer (closed on this pool): every buffer a
kernel writes sits inside a larger allocation whose surrounding guard elements hold a NaN-pattern
canary; after the kernel the canaries must be untouched and the payload must equal the oracle."""
import numpy as np
import pytest

import synth_inputs as si
from oracle import sync
from tests._util import have_gpu, to_dev

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

if have_gpu():
    import torch
    import paper_1706_03292_b200 as pos

CANARY = np.float32(np.frombuffer(np.uint32(0x7FC0DEAD).tobytes(), np.float32)[0])   # a NaN payload


def canary_bits(t):
    return t.view(torch.int32) == int(np.frombuffer(np.float32(CANARY).tobytes(), np.int32)[0])


@pytest.mark.parametrize("dtype", ["bf16", "tf32", "f32"])
@pytest.mark.parametrize("M,N,K,extra_cols", [(129, 260, 8, 4), (65, 36, 8, 8), (300, 520, 32, 4),
                                              (33, 7, 4, 1), (1000, 4100, 16, 12), (7, 1, 1, 3)])
def test_reconstruct_writes_only_its_tile(dtype, M, N, K, extra_cols):
    """W is an M x N window (row stride ldw = N + extra_cols) inside a guarded buffer; the tensor-core
    path is used when ldw % 4 == 0, the SIMT path otherwise."""
    ldw, G0 = N + extra_cols, 64
    P = 2
    Us, Vs = zip(*(si.exact_factors(si.rng(70, 0, p), K, M, N) for p in range(P)))
    W = si.exact_weights(si.rng(71), M, N)
    buf = torch.full((G0 + M * ldw + G0,), float(CANARY), device="cuda")
    Wv = buf[G0:G0 + M * ldw].view(M, ldw)
    Wv[:, :N] = to_dev(W)
    # gather buffer: packed rows for both workers, with its own guards
    R = pos.pos_factor_row_elems(M, N)
    S = pos.pos_factor_slot_rows(K, pos.DTYPES[dtype]) * R      # one worker's slot (f32: 3K rows)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    gbuf = torch.zeros(G0 + P * S + G0, dtype=tdt, device="cuda")
    gbuf[:G0] = 7.0
    gbuf[G0 + P * S:] = 7.0
    for p in range(P):
        slot = gbuf[G0 + p * S: G0 + (p + 1) * S]
        st = "bf16" if dtype == "bf16" else "f32"
        pos.pos_pack_factors(to_dev(Us[p], st), to_dev(Vs[p], st), slot, pos.DTYPES[dtype])
    b = torch.full((M + 2,), float(CANARY), device="cuda")
    bw = si.exact_weights(si.rng(72), M)
    b[1:M + 1] = to_dev(bw)
    pos.pos_reconstruct_apply(M, N, K * P, pos.DTYPES[dtype], gbuf[G0:G0 + P * S], Wv, b[1:M + 1],
                              si.EXACT_ALPHA, ldw=ldw)
    torch.cuda.synchronize()
    assert bool(torch.all(gbuf[:G0] == 7.0)) and bool(torch.all(gbuf[G0 + P * S:] == 7.0))
    assert bool(canary_bits(buf[:G0]).all()) and bool(canary_bits(buf[G0 + M * ldw:]).all())
    if extra_cols:
        assert bool(canary_bits(Wv[:, N:]).all())
    assert bool(canary_bits(b[:1]).all()) and bool(canary_bits(b[M + 1:]).all())
    Wr, br = sync.sfb_update(W, bw, Us, Vs, si.EXACT_ALPHA)
    assert np.array_equal(Wv[:, :N].cpu().numpy().astype(np.float64), Wr)
    assert np.array_equal(b[1:M + 1].cpu().numpy().astype(np.float64), br)


@pytest.mark.parametrize("off,count", [(0, 1), (1, 5), (3, 1001), (0, 4096), (2, 65537)])
def test_ps_apply_writes_only_its_range(off, count):
    G = 32
    g = si.exact_dense_grad(si.rng(73), count)
    w = si.exact_weights(si.rng(74), count)
    Wb = torch.full((G + off + count + G,), float(CANARY), device="cuda")
    gb = torch.full_like(Wb, float(CANARY))
    Wb[G + off:G + off + count] = to_dev(w)
    gb[G + off:G + off + count] = to_dev(g)
    pos.pos_ps_apply(gb[G + off:], Wb[G + off:], count, si.EXACT_ALPHA)
    torch.cuda.synchronize()
    assert bool(canary_bits(Wb[:G + off]).all()) and bool(canary_bits(Wb[G + off + count:]).all())
    assert np.array_equal(Wb[G + off:G + off + count].cpu().numpy().astype(np.float64),
                          sync.ps_update(w, [g], si.EXACT_ALPHA))


@pytest.mark.parametrize("M,N,K", [(13, 7, 5), (21841, 4096, 2), (1, 1, 1)])
def test_pack_writes_only_its_slot(M, N, K):
    R = pos.pos_factor_row_elems(M, N)
    u, v = si.exact_factors(si.rng(75), K, M, N)
    G = 48
    out = torch.full((G + K * R + G,), 3.0, dtype=torch.bfloat16, device="cuda")
    pos.pos_pack_factors(to_dev(u, "bf16"), to_dev(v, "bf16"), out[G:G + K * R], pos.POS_DT_BF16)
    torch.cuda.synchronize()
    assert bool(torch.all(out[:G] == 3.0)) and bool(torch.all(out[G + K * R:] == 3.0))
    slot = out[G:G + K * R].view(K, R).float().cpu().numpy()
    Mp = (M + 63) // 64 * 64
    assert np.array_equal(slot[:, :M], u) and np.array_equal(slot[:, Mp:Mp + N], v)
    assert not slot[:, M:Mp].any() and not slot[:, Mp + N + 1:].any()
    assert np.all(slot[:, Mp + N] == 1.0)          # ones column (fused bias)
