"""Updated-weight definitions for one synchronisation step — fp64, plain numpy.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The method reaches EXACTLY the data-parallel SGD result (it is not an approximation), so the
oracle is that definition written out:

  Eq. 2 (§2.1):  theta(t+1) = theta(t) + eps * sum_{p=1..P} grad_L(theta(t), D_p(t))
  additivity over samples:  the batch gradient is the sum of per-sample gradients
  SFB (§2.1): for an FC layer the per-sample gradient is the rank-1 matrix u v^T,
      u = dL/dy (output gradient, length M), v = x (layer input, length N) [SPEC:300]
  PS  (§2.1): (1) each worker sends its gradient to the servers, (2) servers apply
      (+) the updates to their shard of the parameters, (3) consistency: workers read back.

Readings: S5 alpha carries eps, the sign and any normalisation (W += alpha*G with G
the loss gradient); S6 no 1/P inside the library; S9 shard table from oracle.shard; S11 the
sum order is irrelevant in exact arithmetic; S12 the FC bias gradient is sum_k u_k (the bias
is y = W x + b, so dL/db = dL/dy = u per sample).
"""
from __future__ import annotations

import numpy as np

from .shard import shard_range


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def outer_sum_bruteforce(U, V) -> np.ndarray:
    """sum_k u_k v_k^T with explicit loops. For tiny shapes only."""
    U, V = _f64(U), _f64(V)
    K, M = U.shape
    K2, N = V.shape
    assert K == K2
    G = np.zeros((M, N), dtype=np.float64)
    for k in range(K):
        for i in range(M):
            for j in range(N):
                G[i, j] += U[k, i] * V[k, j]
    return G


def reconstruct(U, V) -> np.ndarray:
    """SFB gradient reconstruction sum_k u_k v_k^T = U^T V (library matmul as one step)."""
    U, V = _f64(U), _f64(V)
    assert U.shape[0] == V.shape[0]
    return U.T @ V


def sfb_update(W, b, Us, Vs, alpha: float):
    """SFB layer after one sync: every worker ends with

        W' = W + alpha * sum_p sum_k u_{p,k} v_{p,k}^T      (Eq. 2 + PAPER:111)
        b' = b + alpha * sum_p sum_k u_{p,k}                (reading S12)

    Us[p]: [K][M] factors u of worker p; Vs[p]: [K][N] factors v of worker p.
    """
    W = _f64(W)
    G = np.zeros_like(W)
    for U, V in zip(Us, Vs):          # sum over workers p (Eq. 2)
        G += reconstruct(U, V)
    W_new = W + alpha * G
    b_new = None
    if b is not None:
        gb = np.zeros(W.shape[0], dtype=np.float64)
        for U in Us:
            gb += _f64(U).sum(axis=0)
        b_new = _f64(b) + alpha * gb
    return W_new, b_new


def ps_update(W_flat, grads, alpha: float):
    """PS layer after one sync (PAPER:107 three steps), through the shard table.

    W_flat: [n] parameters; grads[p]: [n] gradient of worker p. Server r owns shard r
    (oracle.shard), sums the P pushed gradients for its shard, applies (+) them, and every
    worker reads the fresh shard back. Returns the parameters every worker holds.
    """
    W = _f64(W_flat)
    n = W.shape[0]
    P = len(grads)
    out = np.empty_like(W)
    for r in range(P):                                  # each server shard
        lo, hi = shard_range(n, P, r)
        acc = np.zeros(hi - lo, dtype=np.float64)
        for g in grads:                                 # step (1): pushes from every worker
            acc += _f64(g)[lo:hi]
        out[lo:hi] = W[lo:hi] + alpha * acc             # step (2): apply (+)
    return out                                          # step (3): all workers read it back


def fc_grad(U, V) -> np.ndarray:
    """Dense gradient of an FC layer for one worker's batch (what PS pushes for an FC layer)."""
    return reconstruct(U, V)


def wfbp_sync(layers, order=None):
    """Synchronise every layer of one iteration in `order` (default: backward order L..1).

    layers: list of dicts {"scheme": "SFB"|"PS", ...} with the arguments of sfb_update /
    ps_update. WFBP only reschedules the independent s^l, so the result must
    not depend on `order`. Returns a list of per-layer results in layer order.
    """
    L = len(layers)
    order = list(range(L - 1, -1, -1)) if order is None else list(order)
    assert sorted(order) == list(range(L))
    out = [None] * L
    for l in order:
        d = layers[l]
        if d["scheme"] == "SFB":
            out[l] = sfb_update(d["W"], d.get("b"), d["Us"], d["Vs"], d["alpha"])
        else:
            out[l] = ps_update(d["W"], d["grads"], d["alpha"])
    return out
