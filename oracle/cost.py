"""Table 1 cost model and Algorithm 1 (BestScheme) — exact arithmetic.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER:169-183 §3.2 Table 1 ("Estimated communication cost of PS, SFB and Adam for synchronizing
the parameters of a M x N FC layer on a cluster with P1 workers and P2 servers, when batchsize
is K"):

    Method | Server              | Worker          | Server & Worker
    PS     | 2 P1 M N / P2       | 2 M N           | 2 M N (P1 + P2 - 2) / P2
    SFB    | N/A                 | 2 K (P1-1)(M+N) | N/A
    Adam   | P1 M N + P1 K (M+N) | K (M+N) + M N   | (P1 - 1)(M N + K M + K N)

PAPER:217-228 Algorithm 1:
    if layer.type == FC:  if 2K(P1-1)(M+N) <= 2MN(P1+P2-2)/P2: return SFB
    return PS

Readings: S1 the comparison uses the Server&Worker PS column, with P1 = P2 = P in
this build; S2 tie -> SFB ("<="); S3 K = per-worker batch; S4 the division is real-valued —
evaluated here with exact Fractions, no rounding; S7 the formulas are symmetric in (M, N);
S8 P = 1 gives 0 <= 0 -> SFB; S19 only FC layers can be SFB ("indecomposable" CONV/BN -> PS,
PAPER:168 "if l is a CONV layer ... we can directly resort to PS").
"""
from __future__ import annotations

from fractions import Fraction

PS, SFB, ADAM = "PS", "SFB", "ADAM"
SERVER, WORKER, BOTH = "server", "worker", "both"
FC, DENSE = "fc", "dense"


def ps_cost(role: str, M: int, N: int, P1: int, P2: int) -> Fraction:
    """Table 1 row PS."""
    if role == SERVER:
        return Fraction(2 * P1 * M * N, P2)
    if role == WORKER:
        return Fraction(2 * M * N)
    if role == BOTH:
        return Fraction(2 * M * N * (P1 + P2 - 2), P2)
    raise ValueError(role)


def sfb_cost(role: str, M: int, N: int, K: int, P1: int) -> Fraction:
    """Table 1 row SFB. Server / Server&Worker are N/A."""
    if role != WORKER:
        raise ValueError("SFB cost is N/A for role " + role)
    return Fraction(2 * K * (P1 - 1) * (M + N))


def adam_cost(role: str, M: int, N: int, K: int, P1: int) -> Fraction:
    """Table 1 row Adam (max)."""
    if role == SERVER:
        return Fraction(P1 * M * N + P1 * K * (M + N))
    if role == WORKER:
        return Fraction(K * (M + N) + M * N)
    if role == BOTH:
        return Fraction((P1 - 1) * (M * N + K * M + K * N))
    raise ValueError(role)


def cost(scheme: str, role: str, M: int, N: int, K: int, P1: int, P2: int) -> Fraction:
    if scheme == PS:
        return ps_cost(role, M, N, P1, P2)
    if scheme == SFB:
        return sfb_cost(role, M, N, K, P1)
    if scheme == ADAM:
        return adam_cost(role, M, N, K, P1)
    raise ValueError(scheme)


def best_scheme(kind: str, M: int, N: int, K: int, P1: int, P2: int) -> str:
    """Algorithm 1 BestScheme, line by line."""
    # L2-3: layer_property = Query(l.name); P1, P2, K = Query('n_worker','n_server','batchsize')
    if kind == FC:                                   # L4
        # L5-6: M = width, N = height
        if sfb_cost(WORKER, M, N, K, P1) <= ps_cost(BOTH, M, N, P1, P2):   # L7 (exact, real-valued)
            return SFB                               # L8
    return PS                                        # L11


def best_scheme_p(kind: str, M: int, N: int, K: int, P: int) -> str:
    """This build's deployment: every GPU is both a worker and a server shard (P1 = P2 = P, S1)."""
    return best_scheme(kind, M, N, K, P, P)


# ------------------------------------------------------------------------------------------------
# NEXT-3: a B200-calibrated TIME model beside Algorithm 1.
#
# Alg. 1 counts elements on the wire (Table 1) on a 40GbE cluster where the network
# is the only cost. On one NVSwitch box three more things matter (reading S22):
#   * dtypes: SFB factors travel in bf16 (factor_bytes = 2), PS gradients / parameters in fp32;
#   * SFB replicates the update: every GPU reads and writes all of W (8 M N bytes of HBM) and does
#     2 M N K P flops, where PS applies only its shard (12 M N / P bytes: read grad, read W, write W);
#   * PS needs the dense local gradient dW formed first (4 M N bytes written), SFB never forms it.
# Per GPU and iteration, with B_nvl the per-direction NVLink bandwidth and all-to-all traffic
# (every GPU sends and receives the same amount, so one direction bounds):
#   T_SFB = (P-1) K (M+N) fb / B_nvl + max(8 M N / B_hbm, 2 M N K P / F_tc)
#   T_PS  = 2 (P-1)/P * 4 M N / B_nvl + 4 M N / B_hbm + 12 M N / (P B_hbm)
# A bandwidth of None (or 0) drops its terms. Tie -> SFB (as S2).
# Pins (tests/test_oracle_cost.py): with factor_bytes = 4 and the HBM / tensor terms dropped the
# model reduces EXACTLY to Algorithm 1 (the paper's setting: network-only, equal element widths);
# with factor_bytes = 2 (bf16) the SFB region doubles to K (M+N) <= 4 M N / P.
def b200_times(M: int, N: int, K: int, P: int, factor_bytes: int = 2, hbm=6551e9, nvl=770e9,
               tc=1644e12):
    """(T_SFB, T_PS) as exact Fractions of seconds for one FC layer (see the model above)."""
    def inv(x):
        return Fraction(0) if not x else 1 / Fraction(x)
    ihbm, invl, itc = inv(hbm), inv(nvl), inv(tc)
    t_sfb = Fraction((P - 1) * K * (M + N) * factor_bytes) * invl + max(
        Fraction(8 * M * N) * ihbm, Fraction(2 * M * N * K * P) * itc)
    t_ps = Fraction(2 * (P - 1) * 4 * M * N, P) * invl + Fraction(4 * M * N) * ihbm + \
        Fraction(12 * M * N, P) * ihbm
    return t_sfb, t_ps


def b200_time_adam(M: int, N: int, K: int, P: int, factor_bytes: int = 2, hbm=6551e9, nvl=770e9,
                   tc=1644e12):
    """T_ADAM as an exact Fraction of seconds: Table 1's Adam with the layer's rows
    sharded over P owners — SF push (u slice + v to every other owner), the owner's
    reconstruct-and-apply of its M/P rows, matrix pull of the other owners' rows."""
    def inv(x):
        return Fraction(0) if not x else 1 / Fraction(x)
    ihbm, invl, itc = inv(hbm), inv(nvl), inv(tc)
    push = Fraction((P - 1) * K * factor_bytes) * (Fraction(M, P) + N) * invl
    apply = max(Fraction(8 * M * N, P) * ihbm, Fraction(2 * M * N * K) * itc)
    pull = Fraction(4 * (P - 1) * M * N, P) * invl
    return push + apply + pull


def best_scheme_b200(M: int, N: int, K: int, P: int, factor_bytes: int = 2, hbm=6551e9,
                     nvl=770e9, tc=1644e12) -> str:
    t_sfb, t_ps = b200_times(M, N, K, P, factor_bytes, hbm, nvl, tc)
    return SFB if t_sfb <= t_ps else PS
