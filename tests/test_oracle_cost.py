"""Pins for oracle.cost (Table 1, Algorithm 1) against what the paper and the mathematics fix.

Pins used (none re-types the formula under test):
  * the paper's printed worked numbers (tests/golden/paper_pins.txt);
  * an independent message-passing simulator that counts elements per node (oracle.netsim);
  * invariants: monotonicity in K and P, DENSE never SFB, tie -> SFB;
  * the closed form at P1 = P2 = P >= 2:  SFB <=> K P (M+N) <= 2 M N (algebra on Alg. 1 L7).
"""
from fractions import Fraction

import pytest

from oracle import cost, netsim


def _round_sig(x, sig):
    from math import floor, log10
    x = float(x)
    return round(x, -int(floor(log10(abs(x)))) + (sig - 1))


def test_paper_168_vgg_fc_worked_example():
    M = N = 4096
    K, P1, P2 = 32, 8, 8
    w = cost.ps_cost(cost.WORKER, M, N, P1, P2)
    s = cost.ps_cost(cost.SERVER, M, N, P1, P2)
    b = cost.ps_cost(cost.BOTH, M, N, P1, P2)
    f = cost.sfb_cost(cost.WORKER, M, N, K, P1)
    # printed: "approx 34 million", "approx 34 million", "approx 58.7 million", "approx 3.7 million"
    assert _round_sig(w, 2) == 34e6
    assert _round_sig(s, 2) == 34e6
    assert _round_sig(b, 3) == 58.7e6
    assert _round_sig(f, 2) == 3.7e6
    # exact values: integers here
    assert (w, s, b, f) == (33554432, 33554432, 58720256, 3670016)
    assert cost.best_scheme(cost.FC, M, N, K, P1, P2) == cost.SFB


def test_paper_517_googlenet_reduces_to_ps():
    # GoogLeNet's single FC 1000 x 1024, batch 128 (Table 3), 16 nodes each server+worker
    assert cost.best_scheme(cost.FC, 1000, 1024, 128, 16, 16) == cost.PS
    # and at fewer nodes it would have been SFB (the paper's point: the choice depends on P)
    assert cost.best_scheme(cost.FC, 1000, 1024, 128, 4, 4) == cost.SFB


def test_paper_120_alexnet_bandwidth():
    # "240M x 7/8 x 4 = 840M floats": the per-element S&W PS cost at P1 = P2 = 8 is
    # 2(P1+P2-2)/P2 = 3.5 = 4 x 7/8 transfers of each gradient element.
    per_elem = cost.ps_cost(cost.BOTH, 1, 1, 8, 8)
    assert per_elem == Fraction(7, 2) == 4 * Fraction(7, 8)
    floats_per_s = 240_000_000 * per_elem
    assert floats_per_s == 840_000_000
    gbps = floats_per_s * 32 / 1e9
    assert gbps > 26


def test_conv_always_ps():
    for M, N, K, P in [(1, 1, 1, 1), (4096, 4096, 1, 8), (64, 64, 8, 2)]:
        assert cost.best_scheme(cost.DENSE, M, N, K, P, P) == cost.PS


@pytest.mark.parametrize("P1,P2", [(1, 1), (2, 2), (3, 3), (4, 4), (8, 8), (3, 5), (5, 3), (4, 2), (2, 7)])
@pytest.mark.parametrize("M,N", [(2, 3), (4, 4), (6, 10), (12, 5)])
def test_table1_ps_equals_simulated_message_counts(M, N, P1, P2):
    if (M * N) % P2:
        pytest.skip("equal partitioning assumption (PAPER:168) needs P2 | MN for per-role averages")
    # disjoint roles: worker column and server column
    traffic, roles = netsim.simulate_ps(M, N, P1, P2, colocated=False)
    assert netsim.avg_by_role(traffic, roles, {"w"}) == cost.ps_cost(cost.WORKER, M, N, P1, P2)
    assert netsim.avg_by_role(traffic, roles, {"s"}) == cost.ps_cost(cost.SERVER, M, N, P1, P2)
    # co-located roles: the Server & Worker column
    traffic, roles = netsim.simulate_ps(M, N, P1, P2, colocated=True)
    if any(r == {"w", "s"} for r in roles.values()):
        assert netsim.avg_by_role(traffic, roles, {"w", "s"}) == cost.ps_cost(cost.BOTH, M, N, P1, P2)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (4, 3, 2), (7, 5, 3), (8, 8, 4)])
def test_table1_sfb_equals_simulated_message_counts(M, N, K, P):
    t = netsim.simulate_sfb(M, N, K, P)
    for p in range(P):
        assert t[p] == cost.sfb_cost(cost.WORKER, M, N, K, P)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (4, 3, 2), (7, 5, 3), (8, 8, 4), (3, 9, 1)])
def test_ring_collectives_match_table1_with_p1_eq_p2(M, N, K, P):
    """Reading S1: with P1 = P2 = P (every GPU a worker and a shard), ring RS+AG per-rank
    in+out averages to the S&W PS column and ring AG of factor blocks equals the SFB column."""
    rs_ag = netsim.ring_reduce_scatter_allgather(M * N, P)
    assert Fraction(sum(rs_ag), P) == cost.ps_cost(cost.BOTH, M, N, P, P)
    ag = netsim.ring_allgather(K * (M + N), P)
    assert all(x == cost.sfb_cost(cost.WORKER, M, N, K, P) for x in ag)


def test_spec_examples():
    assert cost.sfb_cost(cost.WORKER, 4, 3, 2, 2) == 28
    assert cost.ps_cost(cost.BOTH, 1, 1, 1, 1) == 0
    assert cost.adam_cost(cost.SERVER, 4096, 4096, 32, 8) == 136_314_880
    assert cost.adam_cost(cost.WORKER, 4, 3, 2, 2) == 26
    assert cost.adam_cost(cost.BOTH, 5, 5, 5, 1) == 0


def test_tie_goes_to_sfb():
    # (M,N,K,P) = (2,2,1,2): SFB 2*1*1*4 = 8; PS S&W 2*4*2/2 = 8 -> tie -> SFB ("<=")
    assert cost.sfb_cost(cost.WORKER, 2, 2, 1, 2) == cost.ps_cost(cost.BOTH, 2, 2, 2, 2)
    assert cost.best_scheme(cost.FC, 2, 2, 1, 2, 2) == cost.SFB
    # AlexNet fc7 4096x4096, K=128, P=32: natural tie
    assert cost.sfb_cost(cost.WORKER, 4096, 4096, 128, 32) == cost.ps_cost(cost.BOTH, 4096, 4096, 32, 32)
    assert cost.best_scheme(cost.FC, 4096, 4096, 128, 32, 32) == cost.SFB
    # one more sample flips it
    assert cost.best_scheme(cost.FC, 4096, 4096, 129, 32, 32) == cost.PS


def test_p1_ne_p2_real_division_trap():
    # (M,N,K,P1,P2) = (2,9,1,3,5): SFB 44 vs PS 2*18*6/5 = 43.2 -> PS. A ceil() would say SFB.
    assert cost.sfb_cost(cost.WORKER, 2, 9, 1, 3) == 44
    assert cost.ps_cost(cost.BOTH, 2, 9, 3, 5) == Fraction(216, 5)
    assert cost.best_scheme(cost.FC, 2, 9, 1, 3, 5) == cost.PS


def test_p_equal_1_is_sfb():
    # S8: both costs 0, "0 <= 0" -> SFB (literal Alg. 1)
    for M, N, K in [(1, 1, 1), (64, 64, 8), (21841, 4096, 32)]:
        assert cost.best_scheme(cost.FC, M, N, K, 1, 1) == cost.SFB


def test_grid_invariants_and_closed_form():
    """Tiny grid M,N in [1,16], K in [1,8], P in [1,8]: monotone in K and P,
    closed form at P >= 2: SFB <=> K P (M+N) <= 2MN."""
    for M in range(1, 17):
        for N in range(1, 17):
            for P in range(1, 9):
                prev = cost.SFB
                for K in range(1, 9):
                    s = cost.best_scheme_p(cost.FC, M, N, K, P)
                    if P >= 2:
                        assert (s == cost.SFB) == (K * P * (M + N) <= 2 * M * N)
                    # increasing K never flips PS -> SFB
                    assert not (prev == cost.PS and s == cost.SFB)
                    prev = s
            for K in range(1, 9):
                prev = None
                for P in range(2, 9):
                    s = cost.best_scheme_p(cost.FC, M, N, K, P)
                    assert not (prev == cost.PS and s == cost.SFB)
                    prev = s


def test_grid_counts_survey():
    """SURVEY §8(c) tiny grid M,N in [1,32], K in [1,16], P in [1,16]: 42,300 SFB (16,384 at P=1)
    and 16,575 ties (191 with P > 1). Counts from the survey's independent computation."""
    sfb = ties = ties_p = sfb_p1 = 0
    for M in range(1, 33):
        for N in range(1, 33):
            for K in range(1, 17):
                for P in range(1, 17):
                    f = cost.sfb_cost(cost.WORKER, M, N, K, P)
                    p = cost.ps_cost(cost.BOTH, M, N, P, P)
                    if f <= p:
                        sfb += 1
                        sfb_p1 += P == 1
                    if f == p:
                        ties += 1
                        ties_p += P > 1
    assert (sfb, sfb_p1, ties, ties_p) == (42300, 16384, 16575, 191)


def test_config_schemes():
    """All FC layers of the BASELINE configs are SFB at P in {1,2,4,8}; IncV3 aux FC flips at P=32."""
    from synth_inputs import MODELS, CONFIGS
    for cfg in ("c1", "c2", "c3", "c4"):
        model, K = CONFIGS[cfg]
        for l in MODELS[model].layers:
            for P in (1, 2, 4, 8):
                s = cost.best_scheme_p(l.kind, l.M, l.N, K, P)
                assert s == (cost.SFB if l.kind == "fc" else cost.PS), (cfg, l, P)
    assert cost.best_scheme_p(cost.FC, 1000, 768, 32, 16) == cost.SFB
    assert cost.best_scheme_p(cost.FC, 1000, 768, 32, 32) == cost.PS


# ------------------------------------------------------------------ NEXT-3: B200 time model ----
def test_b200_model_reduces_to_algorithm_1_in_the_papers_setting():
    """Network-only (HBM / tensor terms dropped) and equal element widths (fp32 factors): the B200
    time model must take exactly Alg. 1's decision on every tiny shape."""
    for M in range(1, 13):
        for N in range(1, 13):
            for K in range(1, 9):
                for P in range(1, 9):
                    got = cost.best_scheme_b200(M, N, K, P, factor_bytes=4, hbm=None, tc=None)
                    assert got == cost.best_scheme_p(cost.FC, M, N, K, P), (M, N, K, P)


def test_b200_model_bf16_factors_double_the_sfb_region():
    """bf16 factors vs fp32 PS payload, network only: SFB iff K (M+N) P <= 4 M N (P > 1), i.e.
    twice Alg. 1's K (M+N) P <= 2 M N."""
    for M in range(1, 17):
        for N in range(1, 17):
            for K in range(1, 9):
                for P in range(2, 9):
                    got = cost.best_scheme_b200(M, N, K, P, factor_bytes=2, hbm=None, tc=None)
                    assert got == (cost.SFB if K * (M + N) * P <= 4 * M * N else cost.PS)


def test_b200_model_limits_and_monotonicity():
    # P = 1: no wire; SFB = its replicated apply (8 MN bytes), PS = dW write + full apply (16 MN)
    t_sfb, t_ps = cost.b200_times(4096, 4096, 32, 1, hbm=1.0, nvl=1.0, tc=None)
    assert t_sfb == 8 * 4096 * 4096 and t_ps == 16 * 4096 * 4096
    # larger K only adds to SFB: once PS, always PS
    for (M, N, P) in [(4096, 4096, 8), (1000, 4096, 4), (21841, 4096, 8), (64, 64, 2)]:
        seen_ps = False
        for K in range(1, 2049, 7):
            s = cost.best_scheme_b200(M, N, K, P)
            seen_ps |= s == cost.PS
            assert not (seen_ps and s == cost.SFB), (M, N, P, K)
    # the symmetric formula (reading S7)
    assert cost.b200_times(300, 7000, 64, 8) == cost.b200_times(7000, 300, 64, 8)


def test_b200_model_tensor_term_pinned_to_an_independent_flop_count():
    """The tensor-core term of b200_times (2 M N K P / F_tc) pinned to torch's own flop counter on
    the contraction the method performs: the P workers' K factor rows stacked (Eq. 2) and
    contracted as U^T V. Checked where the term dominates (K P = 2048 > 4 F_tc / B_hbm ~ 1004) and
    where the HBM term does (K P = 64), so a K-vs-K*P slip or a dropped factor 2 fails."""
    import torch
    from torch.utils.flop_counter import FlopCounterMode
    from fractions import Fraction
    hbm, tc = 6551e9, 1644e12
    for (M, N, K, P) in [(96, 160, 256, 8), (4096, 4096, 256, 8), (64, 48, 8, 8)]:
        U = torch.empty(K * P, M, device="meta")
        V = torch.empty(K * P, N, device="meta")
        with FlopCounterMode(display=False) as fc:
            U.t() @ V
        flops = fc.get_total_flops()
        t_sfb, _ = cost.b200_times(M, N, K, P, hbm=hbm, nvl=None, tc=tc)
        t_tc = Fraction(flops) / Fraction(tc)
        t_hbm = Fraction(8 * M * N) / Fraction(hbm)
        assert t_sfb == max(t_tc, t_hbm), (M, N, K, P)
        if K * P > 1004:
            assert t_sfb == t_tc            # tensor-bound regime
        else:
            assert t_sfb == t_hbm


def _adam_bytes_by_enumeration(M, N, K, P, fb):
    """Sharded Adam, transfer by transfer (PAPER:185 'send SFs to a parameter server shard, then
    pull back the whole updated parameter matrices'), rows split into P contiguous equal blocks:
    worker w sends its u rows restricted to owner s's rows and its whole v to every owner s != w;
    owner s sends its W rows (fp32) to every worker w != s. Returns the max over ranks of the bytes
    each rank RECEIVES (the per-direction NVLink volume the model charges)."""
    assert M % P == 0
    rows = M // P
    recv = [0] * P
    for w in range(P):
        for s in range(P):
            if s == w:
                continue
            recv[s] += K * rows * fb + K * N * fb      # SF push: u[:, rows(s)] and v
            recv[w] += rows * N * 4                    # matrix pull: W[rows(s), :]
    return max(recv)


def test_adam_model_pinned_to_transfer_enumeration_and_p1():
    """b200_time_adam: the network term equals the enumerated transfers of the sharded protocol
    (unit bandwidth, no HBM / tensor terms); the apply term equals the owner's share of the
    in-place update (8 bytes per element of its M/P rows); at P = 1 the model is the local
    reconstruct-and-apply, identical to SFB's time."""
    for M in (4, 8, 12):
        for N in (1, 3, 5):
            for K in (1, 2, 7):
                for P in (1, 2, 4):
                    if M % P:
                        continue
                    for fb in (2, 4):
                        net = cost.b200_time_adam(M, N, K, P, fb, hbm=None, nvl=1, tc=None)
                        assert net == _adam_bytes_by_enumeration(M, N, K, P, fb), (M, N, K, P, fb)
                        app = cost.b200_time_adam(M, N, K, P, fb, hbm=1, nvl=None, tc=None)
                        assert app == Fraction(sum(8 * N for _ in range(M // P)))
    for (M, N, K) in [(4096, 4096, 32), (1000, 1024, 128)]:
        t_sfb, _ = cost.b200_times(M, N, K, 1)
        assert cost.b200_time_adam(M, N, K, 1) == t_sfb
