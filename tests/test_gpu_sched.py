"""WFBP scheduler on one GPU (world-1 context): results vs oracle, WFBP == sequential bitwise
(SPEC:369), hazards (WAR on W vs the backward's grad_input read, RAW for the next forward;
PAPER:152), and state-machine misuse -> POS_ESTATE."""
import numpy as np
import pytest

import synth_inputs as si
from oracle import sync
from tests._util import have_gpu, to_dev, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]

if have_gpu():
    import torch
    import paper_1706_03292_b200 as pos

# forward-order layer list: (kind, dims, force_scheme)
LAYERS = [("dense", 1728 + 64, None), ("dense", 2359808, None), ("fc", (4096, 25088, 32), None),
          ("fc", (1000, 4100, 32), pos.POS_SCHEME_PS if have_gpu() else None), ("fc", (21841, 4096, 32), None)]


def make_model(seed):
    """Host arrays: per layer W (+b), the trigger inputs (factors or grad)."""
    out = []
    for l, (kind, dims, force) in enumerate(LAYERS):
        g = si.rng(seed, l)
        if kind == "dense":
            n = dims
            out.append({"kind": kind, "n": n, "W": si.exact_weights(g, n), "g": si.exact_dense_grad(g, n)})
        else:
            M, N, K = dims
            u, v = si.exact_factors(g, K, M, N)
            out.append({"kind": kind, "M": M, "N": N, "K": K, "W": si.exact_weights(g, M, N),
                        "b": si.exact_weights(g, M), "u": u, "v": v, "force": force})
    return out


def oracle_result(model, alpha):
    res = []
    for d in model:
        if d["kind"] == "dense":
            res.append((sync.ps_update(d["W"], [d["g"]], alpha), None))
        else:
            res.append(sync.sfb_update(d["W"], d["b"], [d["u"]], [d["v"]], alpha))
    return res


def run(model, alpha, sequential=False, timing=False, delay_cycles=0, static_tiles=False):
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, len(model), timing=timing, sequential=sequential, static_tiles=static_tiles)
    dev = []
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            n = d["n"]
            P = pos.pos_padded_size(n, 1)
            W = torch.zeros(P, device="cuda"); W[:n] = to_dev(d["W"])
            G = torch.zeros(P, device="cuda"); G[:n] = to_dev(d["g"])
            assert sch.add_dense(l, n, W, G) == pos.POS_SCHEME_PS
            dev.append({"W": W, "G": G})
        else:
            M, N, K = d["M"], d["N"], d["K"]
            if d["force"] == pos.POS_SCHEME_PS:
                n = M * N + M
                P = pos.pos_padded_size(n, 1)
                flat = torch.zeros(P, device="cuda")
                flat[:M * N] = to_dev(d["W"]).reshape(-1)
                flat[M * N:n] = to_dev(d["b"])
                W, b = flat[:M * N].view(M, N), flat[M * N:n]
                grad = torch.empty(P, device="cuda")
                s = sch.add_fc(l, M, N, K, W, b, grad, dtype="bf16", in_dtype=pos.POS_IN_BF16, force_scheme=pos.POS_SCHEME_PS)
                assert s == pos.POS_SCHEME_PS
            else:
                W, b, grad = to_dev(d["W"]), to_dev(d["b"]), None
                s = sch.add_fc(l, M, N, K, W, b, None, dtype="bf16", in_dtype=pos.POS_IN_BF16)
                assert s == pos.POS_SCHEME_SFB  # Alg. 1 at P = 1
            dev.append({"W": W, "b": b, "grad": grad, "u": to_dev(d["u"], "bf16"), "v": to_dev(d["v"], "bf16")})
    for l in range(len(model)):
        assert sch.scheme(l) == (pos.POS_SCHEME_PS if model[l]["kind"] == "dense" or model[l].get("force") == pos.POS_SCHEME_PS else pos.POS_SCHEME_SFB)
    producer = torch.cuda.Stream()
    consumer = torch.cuda.current_stream()
    producer.wait_stream(consumer)
    gi = {}
    sch.begin(alpha)
    with torch.cuda.stream(producer):
        for l in reversed(range(len(model))):            # backward order L..1
            if model[l]["kind"] == "dense":
                sch.grad_ready(l, producer)
            else:
                if delay_cycles:
                    torch.cuda._sleep(delay_cycles)       # a slow b^l
                # b^l reads W: grad_input = grad_output @ W (the WAR hazard the trigger must respect)
                gi[l] = (dev[l]["u"].float() @ dev[l]["W"].float()) if delay_cycles else None
                sch.factors_ready(l, dev[l]["u"], dev[l]["v"], producer)
    sch.end(consumer)
    torch.cuda.synchronize()
    span = sch.timing_span(pos.POS_SCHEME_SFB) if timing and any(
        d["kind"] != "dense" and d.get("force") != pos.POS_SCHEME_PS for d in model) else None
    timings = [sch.timing(l) for l in range(len(model))] if timing else None
    if timing:
        timings = (timings, span)
    out = []
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            out.append((to_host(dev[l]["W"][:d["n"]]), None))
        else:
            out.append((to_host(dev[l]["W"]), to_host(dev[l]["b"])))
    sch.close()
    ctx.close()
    return out, timings, gi


def test_sched_wfbp_matches_oracle_and_sequential_bitwise():
    model = make_model(1)
    a = si.EXACT_ALPHA
    ref = oracle_result(model, a)
    wfbp, _, _ = run(model, a)
    seq, _, _ = run(model, a, sequential=True)
    for (Wr, br), (Ww, bw), (Ws, bs) in zip(ref, wfbp, seq):
        assert np.array_equal(Ww, Wr)
        assert np.array_equal(Ws, Ww)
        if br is not None:
            assert np.array_equal(bw, br) and np.array_equal(bs, bw)


def test_sched_timing_reports():
    model = make_model(2)
    _, (t, span), _ = run(model, si.EXACT_ALPHA, timing=True)
    for pack, comm, apply in t:
        assert pack >= 0 and comm >= 0 and apply > 0
    # the reconstructions' span covers the longest one (they may overlap on two streams)
    sfb = [a for (p, c, a), d in zip(t, model) if d["kind"] != "dense" and d.get("force") != pos.POS_SCHEME_PS]
    if span is not None:
        assert span >= 0.99 * max(sfb)


def test_sched_war_hazard_with_slow_backward():
    """A slow b^l (device sleep) precedes the grad_input read of W; the sync of layer l must not
    touch W before that read (i^l may update only once b^l has finished)."""
    model = make_model(3)
    a = si.EXACT_ALPHA
    out, _, gi = run(model, a, delay_cycles=20_000_000)
    ref = oracle_result(model, a)
    for l, d in enumerate(model):
        assert np.array_equal(out[l][0], ref[l][0])
        if d["kind"] == "fc":
            exp = d["u"].astype(np.float64) @ d["W"].astype(np.float64)   # must see the OLD W
            assert np.array_equal(gi[l].cpu().numpy().astype(np.float64), exp)


def test_sched_misuse_is_estate():
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, 2)
    W = torch.zeros(pos.pos_padded_size(100, 1), device="cuda")
    G = torch.zeros_like(W)
    sch.add_dense(0, 100, W, G)
    with pytest.raises(pos.PoseidonError) as e:
        sch.begin(1.0)                        # layer 1 never added
    assert e.value.code == pos.POS_ESTATE
    sch.add_dense(1, 100, W.clone(), G.clone())
    with pytest.raises(pos.PoseidonError) as e:
        sch.add_dense(1, 100, W, G)           # added twice
    assert e.value.code == pos.POS_ESTATE
    sch.begin(1.0)
    sch.grad_ready(1)
    with pytest.raises(pos.PoseidonError) as e:
        sch.grad_ready(1)                     # triggered twice
    assert e.value.code == pos.POS_ESTATE
    with pytest.raises(pos.PoseidonError) as e:
        sch.end()                             # layer 0 not triggered
    assert e.value.code == pos.POS_ESTATE
    sch.grad_ready(0)
    sch.end()
    with pytest.raises(pos.PoseidonError) as e:
        sch.factors_ready(0, W, W)            # not an FC layer
    assert e.value.code == pos.POS_ESTATE
    torch.cuda.synchronize()
    sch.close()
    ctx.close()


def test_input_validation():
    ctx = pos.Context.local_sim(2)
    W = torch.zeros(64, 64, device="cuda")
    with pytest.raises(pos.PoseidonError) as e:
        pos.lib()  # noqa
        ctx.sync_layer_sfb(torch.zeros(8, 64, device="cuda"), torch.zeros(8, 64, device="cuda"), W)
    assert e.value.code == pos.POS_EINVAL and "pos_sim_sync_layer_sfb" in str(e.value)
    g = torch.zeros(200, device="cuda")
    with pytest.raises(pos.PoseidonError) as e:
        c1 = pos.Context.from_unique_id(bytes(128), 1, 0)
        c1.sync_layer_ps(100, g[1:], g[1:])   # misaligned
    assert e.value.code == pos.POS_EINVAL


def test_sched_cuda_graph_replay_matches_oracle():
    """The scheduler step captured as a CUDA graph (timing on): two replays equal two oracle syncs."""
    model = make_model(4)
    a = si.EXACT_ALPHA
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, len(model), timing=True)
    dev = []
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            n = d["n"]
            P = pos.pos_padded_size(n, 1)
            W = torch.zeros(P, device="cuda"); W[:n] = to_dev(d["W"])
            G = torch.zeros(P, device="cuda"); G[:n] = to_dev(d["g"])
            sch.add_dense(l, n, W, G)
            dev.append({"W": W, "G": G})        # keep G alive: the scheduler holds its pointer
        elif d["force"] is None:
            W, b = to_dev(d["W"]), to_dev(d["b"])
            sch.add_fc(l, d["M"], d["N"], d["K"], W, b, None, dtype="bf16", in_dtype=pos.POS_IN_BF16)
            dev.append({"W": W, "b": b, "u": to_dev(d["u"], "bf16"), "v": to_dev(d["v"], "bf16")})
        else:
            M, N, K = d["M"], d["N"], d["K"]
            n = M * N + M
            flat = torch.zeros(pos.pos_padded_size(n, 1), device="cuda")
            flat[:M * N] = to_dev(d["W"]).reshape(-1)
            flat[M * N:n] = to_dev(d["b"])
            W, b = flat[:M * N].view(M, N), flat[M * N:n]
            grad = torch.empty_like(flat)      # must outlive the scheduler (it keeps the pointer)
            sch.add_fc(l, M, N, K, W, b, grad, dtype="bf16", in_dtype=pos.POS_IN_BF16,
                       force_scheme=pos.POS_SCHEME_PS)
            dev.append({"W": W, "b": b, "grad": grad, "u": to_dev(d["u"], "bf16"), "v": to_dev(d["v"], "bf16")})

    def step(stream):
        sch.begin(a)
        for l in reversed(range(len(model))):
            if model[l]["kind"] == "dense":
                sch.grad_ready(l, stream)
            else:
                sch.factors_ready(l, dev[l]["u"], dev[l]["v"], stream)
        sch.end(stream)

    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
        step(torch.cuda.current_stream())
    torch.cuda.synchronize()
    # capture enqueues nothing: weights unchanged so far
    assert np.array_equal(to_host(dev[0]["W"][:model[0]["n"]]), model[0]["W"].astype(np.float64))
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            r1 = sync.ps_update(d["W"], [d["g"]], a)
            ref = sync.ps_update(r1, [d["g"]], a)
            assert np.array_equal(to_host(dev[l]["W"][:d["n"]]), ref)
        else:
            W1, b1 = sync.sfb_update(d["W"], d["b"], [d["u"]], [d["v"]], a)
            W2, b2 = sync.sfb_update(W1, b1, [d["u"]], [d["v"]], a)
            assert np.array_equal(to_host(dev[l]["W"]), W2)
            assert np.array_equal(to_host(dev[l]["b"]), b2)
    pk, cm, ap = sch.timing(2)          # timing events are real records under replay
    assert ap > 0
    sch.close()
    ctx.close()


@pytest.mark.parametrize("timing", [False, "apply", True])
def test_sched_dense_bucket(timing):
    """Consecutive dense layers synchronised as one bucket (the paper's KV-pair unit): each
    layer's parameters equal the oracle; the bucket is issued only after all its layers trigger."""
    sizes = [1792, 36928, 73856, 5]
    n = sum(sizes)
    a = si.EXACT_ALPHA
    Ws = [si.exact_weights(si.rng(30, i), k) for i, k in enumerate(sizes)]
    Gs = [si.exact_dense_grad(si.rng(31, i), k) for i, k in enumerate(sizes)]
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, len(sizes) + 1, timing=timing)
    Pn = pos.pos_padded_size(n, 1)
    W = torch.zeros(Pn, device="cuda"); W[:n] = to_dev(np.concatenate(Ws))
    G = torch.zeros(Pn, device="cuda"); G[:n] = to_dev(np.concatenate(Gs))
    assert sch.add_dense_bucket(0, sizes, W, G) == pos.POS_SCHEME_PS
    assert len({sch.unit_of(l) for l in range(len(sizes))}) == 1
    Wl = torch.zeros(pos.pos_padded_size(77, 1), device="cuda")
    wl = si.exact_weights(si.rng(32), 77); gl = si.exact_dense_grad(si.rng(33), 77)
    Wl[:77] = to_dev(wl)
    Gl = torch.zeros_like(Wl); Gl[:77] = to_dev(gl)
    sch.add_dense(len(sizes), 77, Wl, Gl)
    sch.begin(a)
    sch.grad_ready(4)
    for l in (3, 2, 1):
        sch.grad_ready(l)
    with pytest.raises(pos.PoseidonError):
        sch.wait_layer(2)                 # bucket not issued yet (layer 0 pending)
    sch.grad_ready(0)
    sch.end()
    torch.cuda.synchronize()
    got = to_host(W[:n])
    off = 0
    for w, g in zip(Ws, Gs):
        assert np.array_equal(got[off:off + len(w)], sync.ps_update(w, [g], a))
        off += len(w)
    assert np.array_equal(to_host(Wl[:77]), sync.ps_update(wl, [gl], a))
    if timing:
        assert sch.timing(0)[2] > 0
    sch.close()
    ctx.close()


@pytest.mark.parametrize("pair", ["0", "1"])
def test_sched_dynamic_tiles_bitwise_equal_static_and_repeatable(pair, monkeypatch):
    """The dynamic tile scheduler (atomic tile fetch, self-resetting counter) changes which CTA
    computes a tile, never the tile's arithmetic: bitwise equal to the static order, over repeated
    iterations (the counter must reset after every launch). pair = "1": the CTA-pair kernel, whose
    leader CTA fetches tiles and broadcasts them to its peer through distributed shared memory."""
    monkeypatch.setenv("POS_SFB_PAIR", pair)
    model = make_model(5)
    a = si.EXACT_ALPHA
    dyn, _, _ = run(model, a)
    sta, _, _ = run(model, a, static_tiles=True)
    for (Wd, bd), (Ws, bs) in zip(dyn, sta):
        assert np.array_equal(Wd, Ws)
    # statistical regime, several iterations: dynamic == static bit for bit
    M, N, K = 4096, 25088, 32
    res = []
    for static in (False, True):
        ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
        sch = pos.Scheduler(ctx, 1, static_tiles=static)
        g = si.rng(60)
        u, v = si.stat_factors(g, K, M, N, "bf16")
        W = to_dev(si.stat_weights(si.rng(61), M, N))
        sch.add_fc(0, M, N, K, W, None, None, "bf16", pos.POS_IN_BF16)
        ud, vd = to_dev(u, "bf16"), to_dev(v, "bf16")
        for _ in range(5):
            sch.begin(-0.01)
            sch.factors_ready(0, ud, vd)
            sch.end()
        torch.cuda.synchronize()
        res.append(W.cpu().numpy())
        sch.close()
        ctx.close()
    assert np.array_equal(res[0], res[1])


def test_sched_wait_layer_raw_gate_per_layer():
    """pos_sched_wait_layer (the per-layer RAW gate for the next forward): a consumer
    stream that waits for ONE layer reads that layer's updated W while another layer's sync is
    still held back behind a slow producer (device sleep before its trigger)."""
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, 2)
    a = si.EXACT_ALPHA
    dims = [(1000, 4100, 16), (4096, 4096, 16)]
    host, dev = [], []
    for l, (M, N, K) in enumerate(dims):
        g = si.rng(70, l)
        u, v = si.exact_factors(g, K, M, N)
        W, b = si.exact_weights(g, M, N), si.exact_weights(g, M)
        host.append((W, b, u, v))
        Wd, bd = to_dev(W), to_dev(b)
        assert sch.add_fc(l, M, N, K, Wd, bd, None, "bf16", pos.POS_IN_BF16) == pos.POS_SCHEME_SFB
        dev.append((Wd, bd, to_dev(u, "bf16"), to_dev(v, "bf16")))
    producer, consumer = torch.cuda.Stream(), torch.cuda.Stream()
    producer.wait_stream(torch.cuda.current_stream())
    consumer.wait_stream(torch.cuda.current_stream())
    sch.begin(a)
    with torch.cuda.stream(producer):
        sch.factors_ready(1, dev[1][2], dev[1][3], producer)     # b^2 done: layer 1 issued now
        torch.cuda._sleep(200_000_000)                          # a slow b^1 (~0.1 s)
        sch.factors_ready(0, dev[0][2], dev[0][3], producer)
    sch.wait_layer(1, consumer)                                 # f^2 of the next iteration
    done1 = torch.cuda.Event()
    with torch.cuda.stream(consumer):
        snap = dev[1][0].clone()                                # reads W^2 after its sync only
        done1.record(consumer)
    done1.synchronize()
    still_running = not producer.query()                        # layer 0 still held back
    sch.end(torch.cuda.current_stream())
    torch.cuda.synchronize()
    W1, b1 = sync.sfb_update(host[1][0], host[1][1], [host[1][2]], [host[1][3]], a)
    W0, b0 = sync.sfb_update(host[0][0], host[0][1], [host[0][2]], [host[0][3]], a)
    assert np.array_equal(to_host(snap), W1)
    assert np.array_equal(to_host(dev[1][0]), W1) and np.array_equal(to_host(dev[0][0]), W0)
    assert np.array_equal(to_host(dev[0][1]), b0)
    assert still_running, "the gate waited for the whole iteration, not for layer 1 only"
    sch.close()
    ctx.close()


def test_factors_ready_rows_must_equal_registered_k():
    """Boundary memory safety: a trigger with fewer (or more) factor rows than the registered K is
    refused with POS_EINVAL instead of letting the pack read past u and v."""
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, 1)
    M, N, K = 256, 512, 16
    W = torch.zeros(M, N, device="cuda")
    sch.add_fc(0, M, N, K, W, None, None, "bf16", pos.POS_IN_BF16)
    u = torch.zeros(K, M, device="cuda", dtype=torch.bfloat16)
    v = torch.zeros(K, N, device="cuda", dtype=torch.bfloat16)
    sch.begin(1.0)
    for rows in (K - 1, K + 1):
        with pytest.raises(pos.PoseidonError) as e:
            sch.factors_ready(0, u[:rows] if rows < K else torch.zeros(rows, M, device="cuda", dtype=torch.bfloat16), v)
        assert e.value.code == pos.POS_EINVAL
    sch.factors_ready(0, u, v)
    sch.end()
    torch.cuda.synchronize()
    sch.close()
    ctx.close()


def test_split_events_pack_before_weights_free():
    """factors_ready / weights_free as separate events (§8(b)): the trigger's weights_free event is
    recorded after a slow grad_input GEMM that reads W; the reconstruction must wait for it (the GEMM
    sees the OLD W) while the result still equals the oracle."""
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, 1, timing=True)
    M, N, K = 4096, 4096, 32
    a = si.EXACT_ALPHA
    g = si.rng(71)
    u, v = si.exact_factors(g, K, M, N)
    W0, b0 = si.exact_weights(g, M, N), si.exact_weights(g, M)
    Wd, bd = to_dev(W0), to_dev(b0)
    sch.add_fc(0, M, N, K, Wd, bd, None, "bf16", pos.POS_IN_BF16)
    ud, vd = to_dev(u, "bf16"), to_dev(v, "bf16")
    producer = torch.cuda.Stream()
    producer.wait_stream(torch.cuda.current_stream())
    ev_f, ev_w = torch.cuda.Event(), torch.cuda.Event()
    sch.begin(a)
    with torch.cuda.stream(producer):
        ev_f.record(producer)
        torch.cuda._sleep(50_000_000)                 # a slow b^l ...
        gi = ud.float() @ Wd                          # ... whose grad_input GEMM reads W
        ev_w.record(producer)
        sch.factors_ready(0, ud, vd, factors_ev=ev_f, weights_free=ev_w)
    sch.end(torch.cuda.current_stream())
    torch.cuda.synchronize()
    Wr, br = sync.sfb_update(W0, b0, [u], [v], a)
    assert np.array_equal(to_host(Wd), Wr) and np.array_equal(to_host(bd), br)
    assert np.array_equal(gi.cpu().numpy().astype(np.float64), u.astype(np.float64) @ W0.astype(np.float64))
    sch.close()
    ctx.close()


def test_sched_wait_host_timeout():
    """pos_sched_wait: a host-side bound on Alg. 2 L8 — POS_ETIMEOUT while a (slow) producer holds
    the iteration back, then success once it completes."""
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, 1)
    n = 4096
    W = torch.zeros(pos.pos_padded_size(n, 1), device="cuda")
    G = torch.ones_like(W)
    sch.add_dense(0, n, W, G)
    producer = torch.cuda.Stream()
    sch.begin(1.0)
    with torch.cuda.stream(producer):
        torch.cuda._sleep(500_000_000)                # ~0.25 s
        sch.grad_ready(0, producer)
    sch.end(torch.cuda.current_stream())
    with pytest.raises(pos.PoseidonError) as e:
        sch.wait(5)
    assert e.value.code == pos.POS_ETIMEOUT
    sch.wait(0)                                       # unbounded: completes
    assert float(W[0]) == 1.0
    sch.close()
    ctx.close()


def test_sched_device_trace():
    """POS_SCHED_TRACE: the apply kernels stamp %globaltimer into device records (no events in the
    streams): every unit reports one launch per iteration with a positive duration, the SFB span of
    a step covers its longest reconstruction, and the results are unchanged (oracle, bitwise) —
    also under CUDA-graph replay."""
    model = make_model(6)
    a = si.EXACT_ALPHA
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, len(model), trace=True)
    dev = []
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            n = d["n"]
            W = torch.zeros(pos.pos_padded_size(n, 1), device="cuda"); W[:n] = to_dev(d["W"])
            G = torch.zeros_like(W); G[:n] = to_dev(d["g"])
            sch.add_dense(l, n, W, G)
            dev.append({"W": W, "G": G})
        else:
            W, b = to_dev(d["W"]), to_dev(d["b"])
            sch.add_fc(l, d["M"], d["N"], d["K"], W, b, None, "bf16", pos.POS_IN_BF16)
            dev.append({"W": W, "b": b, "u": to_dev(d["u"], "bf16"), "v": to_dev(d["v"], "bf16")})

    def step(stream):
        sch.begin(a)
        for l in reversed(range(len(model))):
            if model[l]["kind"] == "dense":
                sch.grad_ready(l, stream)
            else:
                sch.factors_ready(l, dev[l]["u"], dev[l]["v"], stream)
        sch.end(stream)

    step(torch.cuda.current_stream())              # first iteration eager (allocates records)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
        step(torch.cuda.current_stream())
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    durs = []
    for l in range(len(model)):
        avg, last, n = sch.trace(l)
        assert n == 3 and avg > 0 and last > 0, (l, avg, last, n)
        durs.append(avg)
    span, steps = sch.trace_span(pos.POS_SCHEME_SFB)
    assert steps == 3
    sfb = [t for t, d in zip(durs, model) if d["kind"] != "dense"]
    assert span >= 0.99 * max(sfb)
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            r = d["W"]
            for _ in range(3):
                r = sync.ps_update(r, [d["g"]], a)
            assert np.array_equal(to_host(dev[l]["W"][:d["n"]]), r)
        else:
            Wr, br = d["W"], d["b"]
            for _ in range(3):
                Wr, br = sync.sfb_update(Wr, br, [d["u"]], [d["v"]], a)
            assert np.array_equal(to_host(dev[l]["W"]), Wr) and np.array_equal(to_host(dev[l]["b"]), br)
    sch.trace_reset()
    assert sch.trace(0)[2] == 0
    g = None
    sch.close()
    ctx.close()


@pytest.mark.gpu
def test_sched_set_trace_toggle_under_capture():
    """pos_sched_set_trace: a scheduler created untraced runs (eager and captured) iterations, then
    tracing is switched on and the FIRST traced iteration is captured into a CUDA graph (the trace
    records are allocated by set_trace, outside the capture); only the traced replays are counted,
    and the results match the oracle bitwise throughout."""
    model = make_model(6)
    a = si.EXACT_ALPHA
    ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    sch = pos.Scheduler(ctx, len(model), trace=False)
    dev = []
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            n = d["n"]
            W = torch.zeros(pos.pos_padded_size(n, 1), device="cuda"); W[:n] = to_dev(d["W"])
            G = torch.zeros_like(W); G[:n] = to_dev(d["g"])
            sch.add_dense(l, n, W, G)
            dev.append({"W": W, "G": G})
        else:
            W, b = to_dev(d["W"]), to_dev(d["b"])
            sch.add_fc(l, d["M"], d["N"], d["K"], W, b, None, "bf16", pos.POS_IN_BF16)
            dev.append({"W": W, "b": b, "u": to_dev(d["u"], "bf16"), "v": to_dev(d["v"], "bf16")})

    def step(stream):
        sch.begin(a)
        for l in reversed(range(len(model))):
            if model[l]["kind"] == "dense":
                sch.grad_ready(l, stream)
            else:
                sch.factors_ready(l, dev[l]["u"], dev[l]["v"], stream)
        sch.end(stream)

    def capture():
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
            step(torch.cuda.current_stream())
        torch.cuda.current_stream().wait_stream(cs)
        return g

    step(torch.cuda.current_stream())               # untraced, eager
    g0 = capture()                                  # untraced, captured
    g0.replay()
    torch.cuda.synchronize()
    with pytest.raises(pos.PoseidonError):
        sch.trace(0)                                # not tracing
    sch.set_trace(True)
    g1 = capture()                                  # first traced iteration: under capture
    g1.replay()
    g1.replay()
    torch.cuda.synchronize()
    for l in range(len(model)):
        avg, last, n = sch.trace(l)
        assert n == 2 and avg > 0 and last > 0, (l, avg, last, n)
    assert sch.trace_span(pos.POS_SCHEME_SFB)[1] == 2
    sch.set_trace(False)
    g0.replay()                                     # the untraced graph still runs untraced
    torch.cuda.synchronize()
    assert sch.trace(0)[2] == 2
    iters = 5   # eager + g0 replay + g1 x 2 + g0 replay (a capture does not execute)
    for l, d in enumerate(model):
        if d["kind"] == "dense":
            r = d["W"]
            for _ in range(iters):
                r = sync.ps_update(r, [d["g"]], a)
            assert np.array_equal(to_host(dev[l]["W"][:d["n"]]), r)
        else:
            Wr, br = d["W"], d["b"]
            for _ in range(iters):
                Wr, br = sync.sfb_update(Wr, br, [d["u"]], [d["v"]], a)
            assert np.array_equal(to_host(dev[l]["W"]), Wr) and np.array_equal(to_host(dev[l]["b"]), br)
    sch.close()
    ctx.close()
