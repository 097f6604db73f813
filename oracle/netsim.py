"""Message-passing simulator that COUNTS elements per node — an independent pin of Table 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Instead of evaluating the Table 1 formulas, this module plays out the exchanges
the paper describes, message by message, and tallies the elements each node sends and receives
(in + out, reading S13). Tests check the formulas in oracle.cost against these tallies.

  PS ("assume parameters are equally partitioned over all server shards"):
      every worker pushes its M*N gradient, split over the P2 shards, and pulls the fresh
      M*N parameters back; messages between co-located roles (a node that is both worker and
      server talking to itself) do not cross the network.
  SFB (Fig. 2b): every worker sends its K factor pairs (u, v), K*(M+N) elements, to
      each of the other P1-1 workers.
  ring collectives (this build's transport): ring reduce-scatter + ring
      all-gather over P nodes with equal chunks (PS with P1 = P2 = P), and ring all-gather of the
      per-rank factor blocks (SFB).

All tallies are exact Fractions averaged over the nodes of a role (the paper's "equally
partitioned" assumption); totals are integers.
"""
from __future__ import annotations

from collections import defaultdict
from fractions import Fraction


def _equal_parts(total: int, parts: int):
    """Split `total` elements into `parts` contiguous chunks as equally as possible."""
    q, r = divmod(total, parts)
    return [q + (1 if i < r else 0) for i in range(parts)]


def simulate_ps(M: int, N: int, P1: int, P2: int, colocated: bool):
    """Play out one PS iteration. Nodes: workers w0..w{P1-1}, servers s0..s{P2-1}.

    colocated=True places server j on the same node as worker j (j < min(P1,P2)), the
    "Server & Worker" column. Returns (traffic per node dict, node roles dict).
    """
    shard = _equal_parts(M * N, P2)
    node_of = {}
    for p in range(P1):
        node_of[("w", p)] = f"n{p}" if colocated else f"w{p}"
    for j in range(P2):
        node_of[("s", j)] = f"n{j}" if colocated else f"s{j}"
    traffic = defaultdict(int)

    def send(src, dst, elems):
        a, b = node_of[src], node_of[dst]
        if a == b:
            return                       # local hand-off, not on the network
        traffic[a] += elems
        traffic[b] += elems

    for p in range(P1):                   # step (1): push gradient shards
        for j in range(P2):
            send(("w", p), ("s", j), shard[j])
    for j in range(P2):                   # step (3): fresh parameters back to every worker
        for p in range(P1):
            send(("s", j), ("w", p), shard[j])
    roles = defaultdict(set)
    for (kind, _), node in node_of.items():
        roles[node].add(kind)
    return dict(traffic), dict(roles)


def simulate_sfb(M: int, N: int, K: int, P1: int):
    """Every worker sends its K pairs (u in R^M, v in R^N) to every other worker."""
    traffic = defaultdict(int)
    for p in range(P1):
        for q in range(P1):
            if p != q:
                traffic[p] += K * (M + N)
                traffic[q] += K * (M + N)
    return {p: traffic.get(p, 0) for p in range(P1)}


def ring_reduce_scatter_allgather(n: int, P: int):
    """Ring RS then ring AG of an n-element buffer over P ranks; per-rank in+out element tally."""
    chunk = _equal_parts(n, P)
    traffic = [0] * P
    # reduce-scatter: P-1 steps; at step s rank r sends chunk (r - s - 1) mod P to rank r+1
    for s in range(P - 1):
        for r in range(P):
            c = (r - s - 1) % P
            traffic[r] += chunk[c]
            traffic[(r + 1) % P] += chunk[c]
    # all-gather: P-1 steps; at step s rank r forwards chunk (r - s) mod P to rank r+1
    for s in range(P - 1):
        for r in range(P):
            c = (r - s) % P
            traffic[r] += chunk[c]
            traffic[(r + 1) % P] += chunk[c]
    return traffic


def ring_allgather(block: int, P: int):
    """Ring AG of one `block`-element contribution per rank; per-rank in+out tally."""
    traffic = [0] * P
    for s in range(P - 1):
        for r in range(P):
            traffic[r] += block
            traffic[(r + 1) % P] += block
    return traffic


def avg_by_role(traffic: dict, roles: dict, want: set) -> Fraction:
    nodes = [n for n, rs in roles.items() if rs == want]
    assert nodes, (want, roles)
    return Fraction(sum(traffic.get(n, 0) for n in nodes), len(nodes))
