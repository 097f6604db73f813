"""Reading S16: fp32 factors run as 3xTF32 on the tensor cores. CPU checks of the
arithmetic that reading relies on, independent of the CUDA path: the split x = hi + lo with
hi = tf32_rna(x), lo = tf32_rna(x - hi), and the three-term product hi_u hi_v + hi_u lo_v + lo_u hi_v,
against exact (fp64 / Fraction) products — the per-product error bound, the exactness on the
small-integer inputs of the exact regime, and the 1e-5 north_star tolerance on a K*P-term sum."""
from fractions import Fraction

import numpy as np


def tf32_rna(x):
    """fp32 -> tf32 (10 explicit mantissa bits), round to nearest, ties away from zero."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return (((b + 0x1000) & 0xFFFFE000).astype(np.uint32)).view(np.float32)


def split(x):
    x = np.asarray(x, np.float32)
    hi = tf32_rna(x)
    lo = tf32_rna((x - hi).astype(np.float32))
    return hi, lo


def test_tf32_rounding_is_ties_away_and_ten_bits():
    one_ulp = np.float32(2.0 ** -10)
    # exactly halfway between 1 and 1 + 2^-10 rounds away from zero; just below rounds down
    assert tf32_rna(np.float32(1 + 2.0 ** -11)) == np.float32(1 + one_ulp)
    assert tf32_rna(np.float32(-(1 + 2.0 ** -11))) == np.float32(-(1 + one_ulp))
    assert tf32_rna(np.nextafter(np.float32(1 + 2.0 ** -11), np.float32(0))) == np.float32(1)
    g = np.random.default_rng(0)
    x = g.standard_normal(10000).astype(np.float32)
    h = tf32_rna(x)
    assert np.all((h.view(np.uint32) & 0x1FFF) == 0)                     # 13 low bits clear
    assert np.all(np.abs(h - x) <= 2.0 ** -11 * np.abs(x))               # half a tf32 ulp


def test_split_reconstructs_to_2_pow_minus_21():
    g = np.random.default_rng(1)
    x = (g.standard_normal(100000) * np.exp(g.uniform(-20, 20, 100000))).astype(np.float32)
    hi, lo = split(x)
    err = np.abs(hi.astype(np.float64) + lo.astype(np.float64) - x.astype(np.float64))
    assert np.all(err <= 2.0 ** -21 * np.abs(x.astype(np.float64)))


def test_three_term_product_error_bound():
    """|hi_u hi_v + hi_u lo_v + lo_u hi_v - u v| <= 2^-20 |u v| per product (the dropped lo_u lo_v
    term is <= 2^-22 |u v|; the rounding of the two lo parts adds <= 2^-21 each, to first order)."""
    g = np.random.default_rng(2)
    u = g.standard_normal(50000).astype(np.float32)
    v = g.standard_normal(50000).astype(np.float32)
    hu, lu = split(u)
    hv, lv = split(v)
    d = np.float64
    three = hu.astype(d) * hv.astype(d) + hu.astype(d) * lv.astype(d) + lu.astype(d) * hv.astype(d)
    exact = u.astype(d) * v.astype(d)
    assert np.all(np.abs(three - exact) <= 2.0 ** -20 * np.abs(exact))


def test_exact_regime_inputs_split_without_remainder():
    """SURVEY §8(c) exact regime: u in {-4..4}, v in {0..4} — hi = x, lo = 0, so the 3xTF32 rows
    reproduce the plain products bit for bit (the GPU's exact-regime parity stays bitwise)."""
    x = np.arange(-4, 5, dtype=np.float32)
    hi, lo = split(x)
    assert np.array_equal(hi, x) and not np.any(lo)
    ones_hi, ones_lo = split(np.float32([1.0, 0.0]))   # ones column / padding: 1 -> (1, 0), 0 -> (0, 0)
    assert list(ones_hi) == [1.0, 0.0] and list(ones_lo) == [0.0, 0.0]


def test_sum_over_kp_rows_within_north_star_tolerance():
    """A reconstruction column sum over K*P = 1024 statistical-regime products, the three terms
    accumulated in fp32 (as in TMEM): normwise error vs the exact Fraction sum well inside 1e-5."""
    g = np.random.default_rng(3)
    KP, M = 1024, 64
    U = (g.standard_normal((KP, M)) * 2 ** -5).astype(np.float32)
    v = np.maximum(g.standard_normal(KP), 0).astype(np.float32)
    hU, lU = split(U)
    hv, lv = split(v)
    acc = np.zeros(M, np.float32)
    for j in range(KP):   # fp32 accumulation, one term at a time
        acc = (acc + hU[j] * hv[j]).astype(np.float32)
        acc = (acc + hU[j] * lv[j]).astype(np.float32)
        acc = (acc + lU[j] * hv[j]).astype(np.float32)
    exact = np.array([float(sum(Fraction(float(U[j, m])) * Fraction(float(v[j])) for j in range(KP)))
                      for m in range(M)])
    assert np.max(np.abs(acc - exact)) / np.max(np.abs(exact)) <= 1e-5
