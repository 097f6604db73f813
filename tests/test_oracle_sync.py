"""Pins for oracle.sync (updated-weight definitions).

  * brute-force per-sample outer-product loops vs reconstruct (U^T V) — bitwise on ints;
  * closed form u=[1,2], v=[3,4] -> [[3,4],[6,8]];
  * torch CPU autograd of y = x W^T + b: dL/dW == sum_k u_k v_k^T and dL/db == sum_k u_k
    — an independent implementation of the FC gradient;
  * PS through the shard table == plain sum over workers (bitwise on ints, any P);
  * SFB == PS for an FC layer (g_p = U_p^T V_p), bitwise in the exact regime;
  * alpha = 0 and zero factors leave W unchanged; P = 1 is local SGD;
  * WFBP: results independent of layer order.
"""
import numpy as np
import pytest
import torch

import synth_inputs as si
from oracle import sync


def test_closed_form_rank1():
    G = sync.reconstruct(np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]]))
    assert G.tolist() == [[3.0, 4.0], [6.0, 8.0]]


@pytest.mark.parametrize("K,M,N", [(1, 1, 1), (3, 4, 5), (8, 7, 3), (5, 16, 9)])
def test_reconstruct_equals_bruteforce_outer_products(K, M, N):
    g = si.rng(1, K, M)
    U, V = si.exact_factors(g, K, M, N)
    assert np.array_equal(sync.reconstruct(U, V), sync.outer_sum_bruteforce(U, V))
    Us, Vs = si.stat_factors(g, K, M, N, "bf16")
    np.testing.assert_allclose(sync.reconstruct(Us, Vs), sync.outer_sum_bruteforce(Us, Vs), rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("K,M,N", [(1, 3, 2), (8, 64, 64), (4, 10, 33)])
def test_reconstruct_equals_torch_autograd_fc_gradient(K, M, N):
    g = si.rng(2, K, M)
    x = torch.tensor(g.standard_normal((K, N)), dtype=torch.float64)
    W = torch.tensor(g.standard_normal((M, N)), dtype=torch.float64, requires_grad=True)
    b = torch.tensor(g.standard_normal(M), dtype=torch.float64, requires_grad=True)
    R = torch.tensor(g.standard_normal((K, M)), dtype=torch.float64)
    y = torch.nn.functional.linear(x, W, b)
    (y * R).sum().backward()            # dL/dy = R -> u_k = R[k], v_k = x[k]
    U, V = R.numpy(), x.numpy()
    np.testing.assert_allclose(W.grad.numpy(), sync.reconstruct(U, V), rtol=1e-12, atol=1e-12)
    _, b_new = sync.sfb_update(np.zeros((M, N)), np.zeros(M), [U], [V], 1.0)
    np.testing.assert_allclose(b.grad.numpy(), b_new, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_sfb_update_sums_over_workers(P):
    K, M, N = 4, 9, 7
    Us, Vs = zip(*(si.exact_factors(si.rng(3, 0, p), K, M, N) for p in range(P)))
    W = si.exact_weights(si.rng(3, 1), M, N)
    b = si.exact_weights(si.rng(3, 2), M)
    a = si.EXACT_ALPHA
    W1, b1 = sync.sfb_update(W, b, Us, Vs, a)
    # brute force: every sample of every worker contributes its own outer product (Eq. 2 + PAPER:111)
    G = np.zeros((M, N))
    gb = np.zeros(M)
    for p in range(P):
        for k in range(K):
            G += np.outer(Us[p][k].astype(np.float64), Vs[p][k].astype(np.float64))
            gb += Us[p][k]
    assert np.array_equal(W1, W + a * G)
    assert np.array_equal(b1, b + a * gb)


@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("n", [1, 10, 63, 64, 65, 1000, 4097])
def test_ps_update_equals_plain_sum(P, n):
    grads = [si.exact_dense_grad(si.rng(4, n % 97, p), n) for p in range(P)]
    W = si.exact_weights(si.rng(4, 1), n)
    a = si.EXACT_ALPHA
    out = sync.ps_update(W, grads, a)
    assert np.array_equal(out, W.astype(np.float64) + a * np.sum(np.array(grads, dtype=np.float64), axis=0))


@pytest.mark.parametrize("P", [1, 2, 4])
def test_sfb_equals_ps_for_fc_layer(P):
    K, M, N = 8, 64, 64
    Us, Vs = zip(*(si.exact_factors(si.rng(5, 0, p), K, M, N) for p in range(P)))
    W = si.exact_weights(si.rng(5, 1), M, N)
    a = si.EXACT_ALPHA
    W_sfb, _ = sync.sfb_update(W, None, Us, Vs, a)
    grads = [sync.fc_grad(U, V).reshape(-1) for U, V in zip(Us, Vs)]
    W_ps = sync.ps_update(W.reshape(-1), grads, a).reshape(M, N)
    assert np.array_equal(W_sfb, W_ps)
    # statistical regime: equal to rounding
    Us, Vs = zip(*(si.stat_factors(si.rng(6, 0, p), K, M, N) for p in range(P)))
    W = si.stat_weights(si.rng(6, 1), M, N)
    W_sfb, _ = sync.sfb_update(W, None, Us, Vs, -0.01 / P)
    grads = [sync.fc_grad(U, V).reshape(-1) for U, V in zip(Us, Vs)]
    W_ps = sync.ps_update(W.reshape(-1), grads, -0.01 / P).reshape(M, N)
    assert np.max(np.abs(W_sfb - W_ps)) <= 1e-12 * np.max(np.abs(W_sfb))


def test_degenerate_cases():
    K, M, N = 3, 5, 4
    U, V = si.exact_factors(si.rng(7), K, M, N)
    W = si.exact_weights(si.rng(8), M, N)
    b = si.exact_weights(si.rng(9), M)
    W1, b1 = sync.sfb_update(W, b, [U], [V], 0.0)
    assert np.array_equal(W1, W) and np.array_equal(b1, b)
    W2, b2 = sync.sfb_update(W, b, [np.zeros_like(U)], [V], -1.0)
    assert np.array_equal(W2, W) and np.array_equal(b2, b)
    # P = 1: local SGD step W + alpha * dW
    W3, _ = sync.sfb_update(W, None, [U], [V], -0.5)
    assert np.array_equal(W3, W - 0.5 * (U.astype(np.float64).T @ V))


def test_wfbp_order_independence():
    rng = np.random.default_rng(0)
    layers = []
    for l in range(5):
        if l % 2:
            Us, Vs = zip(*(si.exact_factors(si.rng(10, l, p), 3, 6, 5) for p in range(2)))
            layers.append({"scheme": "SFB", "W": si.exact_weights(si.rng(11, l), 6, 5), "b": None,
                           "Us": Us, "Vs": Vs, "alpha": si.EXACT_ALPHA})
        else:
            layers.append({"scheme": "PS", "W": si.exact_weights(si.rng(12, l), 100),
                           "grads": [si.exact_dense_grad(si.rng(13, l, p), 100) for p in range(2)],
                           "alpha": si.EXACT_ALPHA})
    ref = sync.wfbp_sync(layers, order=range(5))
    for _ in range(5):
        out = sync.wfbp_sync(layers, order=rng.permutation(5))
        for a, b in zip(ref, out):
            if isinstance(a, tuple):
                assert np.array_equal(a[0], b[0])
            else:
                assert np.array_equal(a, b)


def test_model_param_counts_match_paper():
    m = si.MODELS
    assert int(m["vgg19"].total_params / 1e6) == 143                                                  # "143M"
    assert int(m["vgg19_22k"].total_params / 1e6) == 229                                              # "229M"
    fc = sum(l.params for l in m["vgg19_22k"].layers if l.kind == "fc")
    assert round(100 * fc / m["vgg19_22k"].total_params) == 91                                         # "91%"
    assert round(m["inception_v3"].total_params / 1e6) == 27                                           # "27M"
    assert abs(m["alexnet"].total_params - 61.5e6) / 61.5e6 < 0.01                                    # "61.5M"
