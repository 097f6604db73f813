"""PS shard table — contiguous equal shards.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER:253 §4.1 "hash the parameters equally to each KV store"; "partition and
distribute model parameters to server nodes as equally as possible". Reading S9:
contiguous shards of stride S = ceil(n / (64 P)) * 64 elements (64 fp32 = 256 B granules);
rank r owns [min(n, r S), min(n, (r+1) S)). The padded buffer holds P*S elements.
"""
from __future__ import annotations


def shard_stride(n: int, P: int) -> int:
    if n < 1 or P < 1:
        raise ValueError((n, P))
    granules = (n + 64 * P - 1) // (64 * P)      # ceil(n / (64 P))
    return granules * 64


def shard_range(n: int, P: int, r: int) -> tuple[int, int]:
    if not 0 <= r < P:
        raise ValueError((r, P))
    S = shard_stride(n, P)
    return min(n, r * S), min(n, (r + 1) * S)


def padded_size(n: int, P: int) -> int:
    return P * shard_stride(n, P)
