"""North-star full-model parity (north_star "VGG19-22K full-model synchronisation
... that matches the oracle"; "229M parameters", "91% ... FC").

This runs bench.py's OWN step — bench.plan_units (bench.DEFAULT_BUCKET_MB dense buckets), bench.register_units,
bench.make_step (every layer triggered in backward order through the WFBP scheduler) and
bench.capture_ring (the 4-graph CUDA-graph ring bench.py replays), in bench.py's order: eager
warm-up steps, then graph replays — on host-generated inputs, and compares EVERY layer's W (and
b) with oracle.sync iterated the same number of times: bitwise in the exact regime, within the
north_star tolerance (W' and dW) in the statistical regime. WFBP and sequential scheduling of the
full model are also compared bit for bit.
"""
import numpy as np
import pytest

import synth_inputs as si
from oracle import sync
from tests._util import err, have_gpu, to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

if have_gpu():
    import torch
    import paper_1706_03292_b200 as pos
    import bench

WARMUP, RING = 3, 4          # bench.py's minimum warm-up, then one replay of each graph of the ring


class HostFill:
    """fill(kind, layer, tensor, role) for bench.register_units with host-generated values; keeps
    the host arrays for the oracle."""

    def __init__(self, regime, K, seed=90, rank=0):
        self.regime, self.K, self.seed, self.rank = regime, K, seed, rank
        self.host = {}

    def gen(self, l, role, rank):
        """Per-(layer, role) stream; weights are the same on every rank, inputs differ by rank."""
        return si.rng(self.seed + 7 * "Wbuvg".index(role), l, rank if role in "uvg" else 0)

    def __call__(self, kind, l, t, role):
        x = self.value(kind, l, tuple(t.shape), role, self.rank)
        self.host[(l, role)] = x
        t.copy_(to_dev(x, "bf16" if t.dtype == torch.bfloat16 else "f32").reshape(t.shape))

    def value(self, kind, l, shape, role, rank):
        g = self.gen(l, role, rank)
        n = int(np.prod(shape))
        if kind == "fc":
            if role == "W":
                M, N = shape
                return si.exact_weights(g, M, N) if self.regime == "exact" else si.stat_weights(g, M, N)
            if role == "b":
                return si.exact_weights(g, n) if self.regime == "exact" else np.zeros(n, np.float32)
            K, D = shape
            if self.regime == "exact":
                u, v = si.exact_factors(g, K, D, D)
            else:
                u, v = si.stat_factors(g, K, D, D, "bf16")
            return u if role == "u" else v
        if role == "W":
            return si.exact_weights(g, n) if self.regime == "exact" else si.stat_weights(g, 1, n)[0] * 0.05
        return si.exact_dense_grad(g, n) if self.regime == "exact" else si.stat_dense_grad(g, n)


def run_model(config, regime, sequential=False, graphs=True, bucket_mb=None):
    bucket_mb = bench.DEFAULT_BUCKET_MB if bucket_mb is None else bucket_mb
    model_name, K = si.CONFIGS[config]
    model = si.load_model(model_name)
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    units = bench.plan_units(model, int(bucket_mb * 2 ** 20 / 4))
    sch = pos.Scheduler(ctx, len(model.layers), timing="apply", sequential=sequential)
    fill = HostFill(regime, K)
    bufs = bench.register_units(pos, ctx, sch, model, units, K, "bf16", fill)
    alpha = si.EXACT_ALPHA if regime == "exact" else -0.01
    main = torch.cuda.current_stream()
    step = bench.make_step(sch, bufs, alpha)
    torch.cuda.synchronize()
    for _ in range(WARMUP):
        step(main)
    n_iter = WARMUP
    ring = None
    if graphs:
        ring = bench.capture_ring(step, main)
        for g in ring:
            g.replay()
        n_iter += len(ring)
    torch.cuda.synchronize()
    out = {}
    for l, bb in enumerate(bufs):
        out[l] = (to_host(bb["W"]), None if bb["kind"] == "dense" or bb["b"] is None else to_host(bb["b"]))
    ring = None
    sch.close()
    ctx.close()
    return model, fill.host, out, n_iter, alpha


def oracle_model(model, host, n_iter, alpha, others=()):
    """oracle.sync iterated n_iter times per layer; `others` = the other ranks' input dicts (their
    factors / gradients join the sum of Eq. 2)."""
    ref = {}
    for l, ly in enumerate(model.layers):
        if ly.kind == "fc":
            W, b = host[(l, "W")], host.get((l, "b"))
            Us = [host[(l, "u")]] + [o[(l, "u")] for o in others]
            Vs = [host[(l, "v")]] + [o[(l, "v")] for o in others]
            for _ in range(n_iter):
                W, b = sync.sfb_update(W, b, Us, Vs, alpha)
            ref[l] = (W, b)
        else:
            W = host[(l, "W")]
            gs = [host[(l, "g")]] + [o[(l, "g")] for o in others]
            for _ in range(n_iter):
                W = sync.ps_update(W, gs, alpha)
            ref[l] = (W, None)
    return ref


@pytest.mark.parametrize("bucket_mb", [None, 64.0, 0.0])   # bench default (16 MiB at P = 1); 64 MiB; one unit per layer
def test_vgg19_22k_bench_step_graph_ring_exact_bitwise(bucket_mb):
    model, host, got, n_iter, alpha = run_model("c3", "exact", bucket_mb=bucket_mb)
    assert model.total_params == 229052817 and len(model.layers) == 19
    ref = oracle_model(model, host, n_iter, alpha)
    for l, ly in enumerate(model.layers):
        assert np.array_equal(got[l][0].reshape(ref[l][0].shape), ref[l][0]), (l, ly.name)
        if ref[l][1] is not None:
            assert np.array_equal(got[l][1], ref[l][1]), (l, ly.name)


def test_vgg19_22k_bench_step_graph_ring_statistical():
    model, host, got, n_iter, alpha = run_model("c3", "stat")
    ref = oracle_model(model, host, n_iter, alpha)
    for l, ly in enumerate(model.layers):
        W0 = host[(l, "W")].astype(np.float64)
        g, r = got[l][0].reshape(ref[l][0].shape), ref[l][0]
        tol = 2e-3 if ly.kind == "fc" else 1e-5          # bf16 factors / fp32 PS path
        assert err(g, r) <= tol, (l, ly.name, err(g, r))
        assert err(g - W0, r - W0) <= tol, (l, ly.name, err(g - W0, r - W0))
        if got[l][1] is not None:
            assert err(got[l][1], ref[l][1]) <= tol


def test_vgg19_22k_wfbp_equals_sequential_bitwise():
    _, _, wfbp, _, _ = run_model("c3", "exact", graphs=False)
    _, _, seq, _, _ = run_model("c3", "exact", sequential=True, graphs=False)
    for l in wfbp:
        assert np.array_equal(wfbp[l][0], seq[l][0]), l
        if wfbp[l][1] is not None:
            assert np.array_equal(wfbp[l][1], seq[l][1]), l


@pytest.mark.parametrize("config", ["c1", "c4"])
def test_other_configs_bench_step_exact_bitwise(config):
    """AlexNet (K = 128) and Inception-V3 (194 layers, 2 SFB FC layers, BN/conv buckets) through the
    same bench step and graph ring."""
    model, host, got, n_iter, alpha = run_model(config, "exact")
    ref = oracle_model(model, host, n_iter, alpha)
    for l, ly in enumerate(model.layers):
        assert np.array_equal(got[l][0].reshape(ref[l][0].shape), ref[l][0]), (config, l, ly.name)
        if ref[l][1] is not None:
            assert np.array_equal(got[l][1], ref[l][1]), (config, l, ly.name)
