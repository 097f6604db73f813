"""Pins for oracle.shard: partition property by brute force, balance, closed form."""
import pytest

from oracle import shard


def test_partition_bruteforce():
    for P in range(1, 9):
        for n in list(range(1, 600)) + [1023, 1024, 1025, 4097, 10000, 2359808]:
            S = shard.shard_stride(n, P)
            assert S % 64 == 0 and S * P >= n and (S - 64) * P < n      # smallest 64-granule stride covering n
            owner = []
            for r in range(P):
                lo, hi = shard.shard_range(n, P, r)
                assert 0 <= lo <= hi <= n
                owner.extend([r] * (hi - lo))
                assert hi - lo <= S
            # disjoint, in rank order, and covering [0, n) exactly once
            assert len(owner) == n
            assert owner == sorted(owner)
            # balance: all non-trailing ranks full, the short ones together miss < 64 P elements
            assert P * S - n < 64 * P


def test_small_layer_leaves_ranks_empty():
    assert shard.shard_stride(10, 8) == 64
    assert shard.shard_range(10, 8, 0) == (0, 10)
    assert all(shard.shard_range(10, 8, r) == (10, 10) for r in range(1, 8))


def test_invalid():
    with pytest.raises(ValueError):
        shard.shard_stride(0, 2)
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)
