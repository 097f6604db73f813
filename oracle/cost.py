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
