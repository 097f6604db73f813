"""C-ABI library (CPU-only checks): it loads, exports every symbol include/poseidon.h declares,
and its pure host functions agree with the oracle BIT-EXACTLY (scheme choice, Table 1 costs,
shard table). No compute calls (no GPU here)."""
import os
import re
from fractions import Fraction

import pytest

import paper_1706_03292_b200 as pos
from oracle import cost, shard

HEADER = __import__("os").path.join(__import__("os").path.dirname(__file__), "..", "include", "poseidon.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pos_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 30
    lib = pos.lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the binding declares exactly the header's functions (same names)
    from paper_1706_03292_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == names


def test_version():
    assert pos.pos_version() == 200


def test_choose_scheme_tiny_grid_bit_exact():
    """Every (M,N,K,P) in M,N in [1,32], K in [1,16], P in [1,16] (262,144 cases) vs Alg. 1 oracle."""
    lib = pos.lib()
    mismatches = 0
    n_sfb = 0
    for M in range(1, 33):
        for N in range(1, 33):
            for K in range(1, 17):
                for P in range(1, 17):
                    got = lib.pos_choose_scheme(M, N, K, P)
                    exp = cost.SFB if 2 * K * (P - 1) * (M + N) * P <= 2 * M * N * (2 * P - 2) else cost.PS
                    n_sfb += got == pos.POS_SCHEME_SFB
                    mismatches += (got == pos.POS_SCHEME_SFB) != (exp == cost.SFB)
    assert mismatches == 0
    assert n_sfb == 42300


def test_choose_scheme_matches_oracle_fraction_form():
    lib = pos.lib()
    for M in range(1, 13):
        for N in range(1, 13):
            for K in range(1, 7):
                for P1 in range(1, 7):
                    for P2 in range(1, 7):
                        for kind in (pos.POS_KIND_FC, pos.POS_KIND_DENSE):
                            got = lib.pos_choose_scheme2(kind, M, N, K, P1, P2)
                            exp = cost.best_scheme(cost.FC if kind == pos.POS_KIND_FC else cost.DENSE,
                                                   M, N, K, P1, P2)
                            assert pos.SCHEME_NAMES[got] == exp, (kind, M, N, K, P1, P2)
    # the ceil() trap of reading S4
    assert pos.pos_choose_scheme2(pos.POS_KIND_FC, 2, 9, 1, 3, 5) == pos.POS_SCHEME_PS


def test_choose_scheme_large_shapes():
    for (M, N, K, P) in [(4096, 4096, 32, 8), (1000, 1024, 128, 16), (21841, 4096, 32, 8),
                         (4096, 25088, 32, 8), (4096, 4096, 128, 32), (4096, 4096, 129, 32),
                         (1 << 30, 1 << 30, 1 << 30, 1 << 20)]:
        got = pos.SCHEME_NAMES[pos.pos_choose_scheme(M, N, K, P)]
        assert got == cost.best_scheme_p(cost.FC, M, N, K, P), (M, N, K, P)


@pytest.mark.parametrize("scheme,role", [(pos.POS_SCHEME_PS, r) for r in range(3)] +
                         [(pos.POS_SCHEME_SFB, pos.POS_ROLE_WORKER)] +
                         [(pos.POS_SCHEME_ADAM, r) for r in range(3)])
def test_cost_elems_exact(scheme, role):
    names = {pos.POS_SCHEME_PS: cost.PS, pos.POS_SCHEME_SFB: cost.SFB, pos.POS_SCHEME_ADAM: cost.ADAM}
    roles = {0: cost.SERVER, 1: cost.WORKER, 2: cost.BOTH}
    for (M, N, K, P1, P2) in [(4096, 4096, 32, 8, 8), (2, 9, 1, 3, 5), (1, 1, 1, 1, 1), (7, 3, 5, 4, 6),
                              (21841, 4096, 32, 8, 8), (1000, 1024, 128, 16, 16)]:
        num, den = pos.pos_cost_elems(scheme, role, M, N, K, P1, P2)
        assert Fraction(num, den) == cost.cost(names[scheme], roles[role], M, N, K, P1, P2)


def test_cost_elems_na_and_errors():
    with pytest.raises(pos.PoseidonError) as e:
        pos.pos_cost_elems(pos.POS_SCHEME_SFB, pos.POS_ROLE_SERVER, 4, 4, 1, 2, 2)
    assert e.value.code == pos.POS_EUNSUPPORTED
    with pytest.raises(pos.PoseidonError) as e:
        pos.pos_choose_scheme(0, 4, 1, 2)
    assert e.value.code == pos.POS_EINVAL and "must be >= 1" in str(e.value)


def test_shard_table_bit_exact():
    lib = pos.lib()
    import ctypes as C
    b, e = C.c_int64(), C.c_int64()
    for P in range(1, 9):
        for n in range(1, 10001):
            S = lib.pos_shard_stride(n, P)
            assert S == shard.shard_stride(n, P)
            assert lib.pos_padded_size(n, P) == P * S
            for r in range(P):
                assert lib.pos_shard_range(n, P, r, C.byref(b), C.byref(e)) == 0
                assert (b.value, e.value) == shard.shard_range(n, P, r)
    assert lib.pos_shard_stride(0, 4) < 0
    assert lib.pos_shard_range(10, 2, 2, C.byref(b), C.byref(e)) == pos.POS_EINVAL


def test_factor_row_layout():
    # M_pad = ceil(M/64)*64; N_pad = ceil((N+1)/64)*64 (128-byte rows, room for the ones column)
    assert pos.pos_factor_row_elems(21841, 4096) == 21888 + 4160
    assert pos.pos_factor_row_elems(1, 1) == 64 + 64
    assert pos.pos_factor_row_elems(64, 64) == 64 + 128
    assert pos.pos_factor_row_elems(13, 7) == 64 + 64
    # 3xTF32 (reading S16): F32 packs three rows per factor pair
    assert pos.pos_factor_slot_rows(32, pos.POS_DT_BF16) == 32
    assert pos.pos_factor_slot_rows(32, pos.POS_DT_TF32) == 32
    assert pos.pos_factor_slot_rows(32, pos.POS_DT_F32) == (32 if os.environ.get("POS_F32_FFMA") == "1" else 96)
    assert pos.lib().pos_factor_slot_rows(1, 7) == pos.POS_EINVAL


def test_b200_time_model_matches_oracle():
    """NEXT-3 chooser: the C time model (double) equals the oracle's exact-Fraction model to
    rounding, and takes the same decision wherever the two times are not within rounding."""
    shapes = [(4096, 4096, 32), (4096, 25088, 32), (21841, 4096, 32), (1000, 4096, 128),
              (4096, 9216, 128), (2048, 1000, 32), (64, 64, 8), (7, 3, 5), (4096, 4096, 512)]
    for (M, N, K) in shapes:
        for P in (1, 2, 4, 8, 16):
            for fb in (2, 4):
                for (hbm, nvl, tc) in [(6551e9, 770e9, 1644e12), (None, 770e9, None),
                                       (6551e9, 900e9, None)]:
                    s, ts, tp = pos.pos_scheme_times_b200(M, N, K, P, fb, hbm, nvl, tc)
                    es, ep = cost.b200_times(M, N, K, P, fb, hbm, nvl, tc)
                    assert abs(ts - float(es)) <= 1e-12 * float(es) + 1e-30
                    assert abs(tp - float(ep)) <= 1e-12 * float(ep) + 1e-30
                    if abs(float(es - ep)) > 1e-9 * float(max(es, ep)):
                        exp = cost.best_scheme_b200(M, N, K, P, fb, hbm, nvl, tc)
                        assert pos.SCHEME_NAMES[s] == exp, (M, N, K, P, fb, hbm, nvl, tc)


def test_b200_time_model_reproduces_algorithm_1():
    """Network-only, fp32 factors: bit-exact Alg. 1 decisions on a tiny grid (ties included —
    both sides are then exactly representable small integers over the same bandwidth)."""
    lib = pos.lib()
    for M in range(1, 17):
        for N in range(1, 17):
            for K in range(1, 9):
                for P in range(1, 9):
                    s, _, _ = pos.pos_scheme_times_b200(M, N, K, P, 4, 0, 1.0, 0)
                    assert s == lib.pos_choose_scheme(M, N, K, P), (M, N, K, P)


def test_adam_time_model_matches_oracle():
    """Table 1's third scheme in the B200 model: C (double) equals the oracle's exact Fraction."""
    for (M, N, K) in [(4096, 4096, 32), (4096, 25088, 32), (1000, 1024, 128), (7, 3, 5), (64, 64, 8)]:
        for P in (1, 2, 3, 4, 8):
            for fb in (2, 4):
                for (hbm, nvl, tc) in [(6551e9, 770e9, 1644e12), (None, 1.0, None), (6551e9, None, None)]:
                    t = pos.pos_scheme_time_adam_b200(M, N, K, P, fb, hbm, nvl, tc)
                    e = cost.b200_time_adam(M, N, K, P, fb, hbm, nvl, tc)
                    assert abs(t - float(e)) <= 1e-12 * float(e) + 1e-30, (M, N, K, P, fb)
