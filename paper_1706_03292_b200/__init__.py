"""paper_1706_03292_b200 — B200-native Poseidon per-layer gradient synchronisation.

Thin Python binding over libposeidon.so (include/poseidon.h). Names follow the C ABI
(`pos_choose_scheme`, `pos_sync_layer_sfb`, ...); the classes below only marshal torch tensors to
raw device pointers and CUDA stream handles. Every step of the synchronisation runs in the
library's CUDA kernels and NCCL calls; there is no CPU fallback.

Paper: Zhang et al., "Poseidon", USENIX ATC'17 (arXiv 1706.03292).
"""
from __future__ import annotations

import ctypes as C

from ._lib import lib, LIB_PATH

POS_SCHEME_PS, POS_SCHEME_SFB, POS_SCHEME_ADAM = 0, 1, 2
POS_KIND_FC, POS_KIND_DENSE = 0, 1
POS_ROLE_SERVER, POS_ROLE_WORKER, POS_ROLE_BOTH = 0, 1, 2
POS_DT_BF16, POS_DT_TF32, POS_DT_F32 = 0, 1, 2
POS_IN_BF16, POS_IN_F32 = 0, 1
POS_OK, POS_EINVAL, POS_ESTATE, POS_ECUDA, POS_ENCCL, POS_ENOMEM, POS_EUNSUPPORTED = 0, -1, -2, -3, -4, -5, -6
POS_ETIMEOUT = -7
POS_REDUCE_SWITCH, POS_REDUCE_RANK_ORDER, POS_REDUCE_AUTO = 0, 1, 2
POS_FAULT_NONE, POS_FAULT_SKIP_PS, POS_FAULT_SKIP_PACK = 0, 1, 2
POS_SCHED_TIMING, POS_SCHED_SEQUENTIAL, POS_SCHED_TIMING_APPLY, POS_SCHED_NO_SYMM, POS_SCHED_PS_AFTER_SFB = 1, 2, 4, 8, 16
POS_SCHED_STATIC_TILES, POS_SCHED_TRACE = 32, 64

DTYPES = {"bf16": POS_DT_BF16, "tf32": POS_DT_TF32, "f32": POS_DT_F32}
SCHEME_NAMES = {POS_SCHEME_PS: "PS", POS_SCHEME_SFB: "SFB", POS_SCHEME_ADAM: "ADAM"}


class PoseidonError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().pos_last_error().decode(errors="replace")
        super().__init__(f"{where} -> {code}: {msg}")
        self.code = code


def _chk(rc: int, where: str) -> int:
    if rc < 0:
        raise PoseidonError(rc, where)
    return rc


# ------------------------------------------------------------------ pure host functions ----
def pos_version() -> int:
    return lib().pos_version()


def pos_scheme_times_b200(M, N, K, P, factor_bytes=2, hbm=6551e9, nvl=770e9, tc=1644e12):
    """NEXT-3 B200 time model beside Algorithm 1: (scheme, T_SFB seconds, T_PS seconds); a
    bandwidth / flop rate of 0 or None drops its terms (include/poseidon.h)."""
    a, b = C.c_double(), C.c_double()
    r = lib().pos_scheme_times_b200(M, N, K, P, factor_bytes, float(hbm or 0), float(nvl or 0),
                                    float(tc or 0), C.byref(a), C.byref(b))
    _chk(r, "pos_scheme_times_b200")
    return r, a.value, b.value


def pos_scheme_time_adam_b200(M, N, K, P, factor_bytes=2, hbm=6551e9, nvl=770e9, tc=1644e12):
    """Table 1's Adam scheme (SF push to row-sharded owners, matrix pull) in the B200 time model:
    T_ADAM seconds (include/poseidon.h)."""
    t = C.c_double()
    _chk(lib().pos_scheme_time_adam_b200(M, N, K, P, factor_bytes, float(hbm or 0), float(nvl or 0),
                                         float(tc or 0), C.byref(t)), "pos_scheme_time_adam_b200")
    return t.value


def pos_choose_scheme(M: int, N: int, K: int, P: int) -> int:
    return _chk(lib().pos_choose_scheme(M, N, K, P), "pos_choose_scheme")


def pos_choose_scheme2(kind: int, M: int, N: int, K: int, P1: int, P2: int) -> int:
    return _chk(lib().pos_choose_scheme2(kind, M, N, K, P1, P2), "pos_choose_scheme2")


def pos_cost_elems(scheme: int, role: int, M: int, N: int, K: int, P1: int, P2: int):
    """Table 1 cost as an exact (numerator, denominator) pair."""
    num, den = C.c_uint64(), C.c_uint64()
    _chk(lib().pos_cost_elems(scheme, role, M, N, K, P1, P2, C.byref(num), C.byref(den)),
         "pos_cost_elems")
    return num.value, den.value


def pos_shard_stride(n: int, P: int) -> int:
    return _chk(lib().pos_shard_stride(n, P), "pos_shard_stride")


def pos_shard_range(n: int, P: int, r: int):
    b, e = C.c_int64(), C.c_int64()
    _chk(lib().pos_shard_range(n, P, r, C.byref(b), C.byref(e)), "pos_shard_range")
    return b.value, e.value


def pos_padded_size(n: int, P: int) -> int:
    return _chk(lib().pos_padded_size(n, P), "pos_padded_size")


def pos_factor_row_elems(M: int, N: int) -> int:
    return _chk(lib().pos_factor_row_elems(M, N), "pos_factor_row_elems")


def pos_factor_slot_rows(K: int, dtype: int) -> int:
    return _chk(lib().pos_factor_slot_rows(K, dtype), "pos_factor_slot_rows")


# --------------------------------------------------------------------- torch marshalling ----
def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _in_dtype(t):
    import torch
    if t.dtype == torch.bfloat16:
        return POS_IN_BF16
    if t.dtype == torch.float32:
        return POS_IN_F32
    raise TypeError(f"factors must be bf16 or fp32, got {t.dtype}")


def _check_factors(u, v, W):
    assert u.is_cuda and v.is_cuda and W.is_cuda, "tensors must live on the GPU"
    assert u.is_contiguous() and v.is_contiguous() and W.is_contiguous()
    assert u.dtype == v.dtype and W.dtype.is_floating_point and W.element_size() == 4
    K, M = u.shape
    K2, N = v.shape
    assert K == K2 and (tuple(W.shape[-2:]) == (M, N) or W.numel() >= M * N)
    return M, N, K


def pos_pack_factors(u, v, slot, dtype: int, stream=None):
    K, M = u.shape
    N = v.shape[1]
    _chk(lib().pos_pack_factors(M, N, K, _in_dtype(u), dtype, _ptr(u), _ptr(v), _ptr(slot),
                                _stream(stream)), "pos_pack_factors")


def pos_reconstruct_apply(M, N, KP, dtype, G, W, b=None, alpha=1.0, accumulate=True, ldw=None,
                          stream=None):
    _chk(lib().pos_reconstruct_apply(M, N, KP, dtype, _ptr(G), int(accumulate), _ptr(W),
                                     N if ldw is None else ldw, _ptr(b), alpha, _stream(stream)),
         "pos_reconstruct_apply")


def pos_ps_apply(g, W, count, alpha, stream=None):
    _chk(lib().pos_ps_apply(_ptr(g), _ptr(W), count, alpha, _stream(stream)), "pos_ps_apply")


class Context:
    """pos_ctx: NCCL communicator + comm stream + workspace, on the current CUDA device."""

    def __init__(self, handle, world, rank, local):
        self.h = handle
        self.world, self.rank, self.local = world, rank, local

    # construction ---------------------------------------------------------------------
    @classmethod
    def local_sim(cls, P: int = 1) -> "Context":
        h = C.c_void_p()
        _chk(lib().pos_init_local(P, C.byref(h)), "pos_init_local")
        return cls(h, P, 0, True)

    @classmethod
    def from_unique_id(cls, uid: bytes, world: int, rank: int) -> "Context":
        h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        _chk(lib().pos_init(buf, world, rank, C.byref(h)), "pos_init")
        return cls(h, world, rank, False)

    @classmethod
    def from_torch_distributed(cls, group=None) -> "Context":
        """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it (plumbing only)."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        if world == 1:
            return cls.from_unique_id(bytes(128), 1, 0)
        uid = C.create_string_buffer(128)
        if rank == 0:
            _chk(lib().pos_get_unique_id(uid), "pos_get_unique_id")
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).to(dev)
        dist.broadcast(t, src=0, group=group)
        return cls.from_unique_id(bytes(t.cpu().tolist()), world, rank)

    def close(self):
        """pos_finalize. With world > 1 this is COLLECTIVE (NCCL window deregistration and
        communicator teardown): every rank must call it explicitly, in the same order."""
        if self.h:
            _chk(lib().pos_finalize(self.h), "pos_finalize")
            self.h = None

    def __del__(self):
        # No collective teardown from the garbage collector (its order differs across ranks): a
        # multi-rank context that was not closed explicitly is leaked with a warning.
        if getattr(self, "h", None):
            if self.world > 1 and not self.local:
                import warnings
                warnings.warn("poseidon Context (world > 1) garbage-collected without close(): leaked")
                return
            try:
                self.close()
            except Exception:
                pass

    def async_error(self) -> int:
        return lib().pos_get_async_error(self.h)

    def set_max_ctas(self, n: int):
        _chk(lib().pos_set_max_ctas(self.h, n), "pos_set_max_ctas")

    def set_timeout_ms(self, ms: int):
        """Watchdog budget of every cross-GPU wait in the library's kernels (0 = unbounded)."""
        _chk(lib().pos_set_timeout_ms(self.h, int(ms)), "pos_set_timeout_ms")

    def set_reduce_order(self, order: int):
        """POS_REDUCE_SWITCH (NVLS multimem reduce), POS_REDUCE_RANK_ORDER (deterministic) or
        POS_REDUCE_AUTO (default: rank-order peer loads + peer stores at P = 2, else SWITCH)."""
        _chk(lib().pos_set_reduce_order(self.h, order), "pos_set_reduce_order")

    def inject_fault(self, kind: int, rank: int):
        _chk(lib().pos_inject_fault(self.h, kind, rank), "pos_inject_fault")

    def sym_empty(self, numel: int, dtype=None):
        """A zero-filled fp32 torch tensor in symmetric (NVLS multicast) memory — pos_mem_alloc.
        COLLECTIVE: all ranks call it with the same size in the same order. Freed with the context."""
        import torch
        dtype = torch.float32 if dtype is None else dtype
        nbytes = numel * torch.empty(0, dtype=dtype).element_size()
        p = C.c_void_p()
        _chk(lib().pos_mem_alloc(self.h, nbytes, C.byref(p)), "pos_mem_alloc")

        class _Holder:
            __cuda_array_interface__ = {"shape": (numel,), "typestr": {torch.float32: "<f4", torch.bfloat16: "<V2"}.get(dtype, "<f4"),
                                        "data": (p.value, False), "version": 3}
        t = torch.as_tensor(_Holder(), device=torch.device("cuda", torch.cuda.current_device()))
        if dtype != torch.float32:
            t = t.view(dtype)
        t._pos_ctx = self   # the window lives as long as the context: keep the context alive
        return t

    def is_symmetric(self, t) -> bool:
        return bool(lib().pos_mem_is_symmetric(self.h, C.c_void_p(t.data_ptr()), t.numel() * t.element_size()))

    # one-shot syncs ---------------------------------------------------------------------
    def sync_layer_sfb(self, u, v, W, b=None, alpha=1.0, dtype="bf16", stream=None):
        """pos_sync_layer_sfb: W += alpha * sum over all ranks' samples of u v^T (and b += alpha * sum u)."""
        M, N, K = _check_factors(u, v, W)
        _chk(lib().pos_sync_layer_sfb(self.h, M, N, K, _in_dtype(u), DTYPES[dtype], _ptr(u), _ptr(v),
                                      _ptr(W), _ptr(b), alpha, _stream(stream)), "pos_sync_layer_sfb")

    def sync_layer_ps(self, n, grad, W, alpha=1.0, stream=None):
        """pos_sync_layer_ps: grad and W are flat fp32 buffers of >= pos_padded_size(n, P)."""
        assert grad.numel() >= pos_padded_size(n, self.world) and W.numel() >= pos_padded_size(n, self.world)
        _chk(lib().pos_sync_layer_ps(self.h, n, _ptr(grad), _ptr(W), alpha, _stream(stream)),
             "pos_sync_layer_ps")

    def sync_layer_fc_ps(self, u, v, grad, Wb, has_bias, alpha=1.0, dtype="bf16", stream=None):
        K, M = u.shape
        N = v.shape[1]
        _chk(lib().pos_sync_layer_fc_ps(self.h, M, N, K, _in_dtype(u), DTYPES[dtype], _ptr(u), _ptr(v),
                                        _ptr(grad), _ptr(Wb), int(has_bias), alpha, _stream(stream)),
             "pos_sync_layer_fc_ps")

    def sim_sync_layer_sfb(self, us, vs, W, b=None, alpha=1.0, dtype="bf16", stream=None):
        assert self.local and len(us) == len(vs) == self.world
        M, N, K = _check_factors(us[0], vs[0], W)
        up = (C.c_void_p * len(us))(*[u.data_ptr() for u in us])
        vpp = (C.c_void_p * len(vs))(*[v.data_ptr() for v in vs])
        _chk(lib().pos_sim_sync_layer_sfb(self.h, M, N, K, _in_dtype(us[0]), DTYPES[dtype], up, vpp,
                                          _ptr(W), _ptr(b), alpha, _stream(stream)),
             "pos_sim_sync_layer_sfb")

    def loop_sync_layer_ps(self, n, grads, Ws, alpha=1.0, stream=None):
        """pos_loop_sync_layer_ps: P simulated ranks' replicas (flat fp32, >= pos_padded_size(n, P))."""
        assert self.local and len(grads) == len(Ws) == self.world
        gp = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        wp = (C.c_void_p * len(Ws))(*[w.data_ptr() for w in Ws])
        _chk(lib().pos_loop_sync_layer_ps(self.h, n, gp, wp, alpha, _stream(stream)), "pos_loop_sync_layer_ps")

    def loop_sync_layer_ps_ce(self, n, grads, Ws, alpha=1.0, stream=None):
        """pos_loop_sync_layer_ps_ce: the copy-engine PS unit's kernels over P simulated replicas."""
        assert self.local and len(grads) == len(Ws) == self.world
        gp = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        wp = (C.c_void_p * len(Ws))(*[w.data_ptr() for w in Ws])
        _chk(lib().pos_loop_sync_layer_ps_ce(self.h, n, gp, wp, alpha, _stream(stream)),
             "pos_loop_sync_layer_ps_ce")

    def sim_sync_layer_ps(self, grads, W, alpha=1.0, n=None, stream=None):
        assert self.local and len(grads) == self.world
        n = W.numel() if n is None else n
        gp = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        _chk(lib().pos_sim_sync_layer_ps(self.h, n, gp, _ptr(W), alpha, _stream(stream)),
             "pos_sim_sync_layer_ps")


class LoopFC:
    """pos_loop_fc: a loopback FC layer with one replica of W (and b) per simulated rank."""

    def __init__(self, ctx: Context, M, N, K, Ws, bs=None, dtype="bf16"):
        assert ctx.local and len(Ws) == ctx.world
        self.ctx, self.M, self.N, self.K = ctx, M, N, K
        self._keep = (list(Ws), None if bs is None else list(bs))
        wp = (C.c_void_p * len(Ws))(*[w.data_ptr() for w in Ws])
        bp = None if bs is None else (C.c_void_p * len(bs))(*[b.data_ptr() for b in bs])
        h = C.c_void_p()
        _chk(lib().pos_loop_fc_create(ctx.h, M, N, K, DTYPES[dtype], wp, bp, C.byref(h)), "pos_loop_fc_create")
        self.h = h

    def sync(self, us, vs, alpha, stream=None):
        up = (C.c_void_p * len(us))(*[u.data_ptr() for u in us])
        vp_ = (C.c_void_p * len(vs))(*[v.data_ptr() for v in vs])
        _chk(lib().pos_loop_fc_sync(self.h, _in_dtype(us[0]), up, vp_, alpha, _stream(stream)), "pos_loop_fc_sync")

    def close(self):
        if self.h:
            lib().pos_loop_fc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Scheduler:
    """pos_sched: WFBP per-layer scheduler (Algorithm 2 on CUDA streams/events)."""

    def __init__(self, ctx: Context, n_layers: int, timing=False, sequential=False, symm=True,
                 ps_after_sfb=False, static_tiles=False, trace=False):
        """timing: False | True (all stages) | "apply" (apply stage only). symm: place SFB gather
        buffers in symmetric memory (multicast factor pack) when world > 1."""
        self.ctx = ctx
        h = C.c_void_p()
        tflag = POS_SCHED_TIMING_APPLY if timing == "apply" else (POS_SCHED_TIMING if timing else 0)
        flags = (tflag | (POS_SCHED_SEQUENTIAL if sequential else 0) | (0 if symm else POS_SCHED_NO_SYMM)
                 | (POS_SCHED_PS_AFTER_SFB if ps_after_sfb else 0) | (POS_SCHED_STATIC_TILES if static_tiles else 0)
                 | (POS_SCHED_TRACE if trace else 0))
        _chk(lib().pos_sched_create(ctx.h, n_layers, flags, C.byref(h)), "pos_sched_create")
        self.h = h
        self.L = n_layers
        self._ev = {}        # one cached CUDA event per (layer, role): trigger plumbing only

    def add_fc(self, l, M, N, K, W, b=None, grad=None, dtype="bf16", in_dtype=POS_IN_BF16, force_scheme=-1):
        return _chk(lib().pos_sched_add_fc(self.h, l, M, N, K, in_dtype, DTYPES[dtype], _ptr(W), _ptr(b),
                                           _ptr(grad), force_scheme), "pos_sched_add_fc")

    def add_dense(self, l, n, W, grad):
        return _chk(lib().pos_sched_add_dense(self.h, l, n, _ptr(W), _ptr(grad)), "pos_sched_add_dense")

    def add_dense_bucket(self, l_first, sizes, W, grad):
        """Consecutive dense layers l_first.. stored back to back in W / grad (flat fp32)."""
        arr = (C.c_int64 * len(sizes))(*sizes)
        return _chk(lib().pos_sched_add_dense_bucket(self.h, l_first, len(sizes), arr, _ptr(W), _ptr(grad)),
                    "pos_sched_add_dense_bucket")

    def unit_of(self, l):
        return _chk(lib().pos_sched_unit_of(self.h, l), "pos_sched_unit_of")

    def begin(self, alpha):
        _chk(lib().pos_sched_begin(self.h, alpha), "pos_sched_begin")

    def _event(self, key, stream):
        """Record this (layer, role)'s cached event on `stream` and return its handle."""
        import torch
        ev = self._ev.get(key)
        if ev is None:
            ev = self._ev[key] = torch.cuda.Event()
        ev.record(torch.cuda.current_stream() if stream is None else stream)
        return C.c_void_p(ev.cuda_event)

    def factors_ready(self, l, u, v, stream=None, factors_ev=None, weights_free=None):
        """pos_sched_factors_ready. Events are torch.cuda.Event objects already recorded by the
        caller; if factors_ev is None, an event is recorded on `stream` now (then the pack also
        waits for everything enqueued on it so far). weights_free=None: same as factors_ready."""
        fe = C.c_void_p(factors_ev.cuda_event) if factors_ev is not None else self._event((l, 0), stream)
        we = None if weights_free is None else C.c_void_p(weights_free.cuda_event)
        _chk(lib().pos_sched_factors_ready(self.h, l, u.shape[0], _ptr(u), _ptr(v), fe, we),
             "pos_sched_factors_ready")

    def grad_ready(self, l, stream=None, event=None):
        ge = C.c_void_p(event.cuda_event) if event is not None else self._event((l, 1), stream)
        _chk(lib().pos_sched_grad_ready(self.h, l, ge), "pos_sched_grad_ready")

    def wait(self, timeout_ms=0):
        """pos_sched_wait: host wait for the last iteration with a timeout (eager mode)."""
        _chk(lib().pos_sched_wait(self.h, int(timeout_ms)), "pos_sched_wait")

    def wait_layer(self, l, stream=None):
        _chk(lib().pos_sched_wait_layer(self.h, l, _stream(stream)), "pos_sched_wait_layer")

    def end(self, stream=None):
        _chk(lib().pos_sched_end(self.h, _stream(stream)), "pos_sched_end")

    def end_layers(self, stream=None):
        """pos_sched_end_layers: close the iteration; consumers gate per layer with wait_layer."""
        _chk(lib().pos_sched_end_layers(self.h, _stream(stream)), "pos_sched_end_layers")

    def scheme(self, l):
        return _chk(lib().pos_sched_scheme(self.h, l), "pos_sched_scheme")

    def timing(self, l):
        a, b, c = C.c_float(), C.c_float(), C.c_float()
        _chk(lib().pos_sched_timing(self.h, l, C.byref(a), C.byref(b), C.byref(c)), "pos_sched_timing")
        return a.value, b.value, c.value

    def timeline(self, n_units):
        """pos_sched_timeline: per unit [start, packed, gathered, apply0, apply1, done] in ms."""
        buf = (C.c_float * (6 * n_units))()
        n = _chk(lib().pos_sched_timeline(self.h, buf, n_units), "pos_sched_timeline")
        return [list(buf[6 * u:6 * u + 6]) for u in range(min(n, n_units))]

    def trace(self, l):
        """pos_sched_trace: (average us, last us, launches) of layer l's unit apply kernel."""
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        _chk(lib().pos_sched_trace(self.h, l, C.byref(a), C.byref(b), C.byref(n)), "pos_sched_trace")
        return a.value, b.value, n.value

    def trace_last(self, l):
        """pos_sched_trace_last: (start_ns, end_ns) %globaltimer stamps of layer l's last traced launch."""
        a, b = C.c_int64(), C.c_int64()
        _chk(lib().pos_sched_trace_last(self.h, l, C.byref(a), C.byref(b)), "pos_sched_trace_last")
        return a.value, b.value

    def trace_span(self, scheme=None):
        """pos_sched_trace_span: (average us, steps) of the step's apply-kernel span of `scheme`."""
        a, n = C.c_double(), C.c_int64()
        _chk(lib().pos_sched_trace_span(self.h, POS_SCHEME_SFB if scheme is None else scheme,
                                        C.byref(a), C.byref(n)), "pos_sched_trace_span")
        return a.value, n.value

    def trace_reset(self):
        _chk(lib().pos_sched_trace_reset(self.h), "pos_sched_trace_reset")

    def set_trace(self, on):
        """pos_sched_set_trace: device-side tracing on / off for the iterations issued from now on."""
        _chk(lib().pos_sched_set_trace(self.h, 1 if on else 0), "pos_sched_set_trace")

    def timing_reset(self):
        _chk(lib().pos_sched_timing_reset(self.h), "pos_sched_timing_reset")

    def timing_span(self, scheme=None):
        """Device ms from the earliest to the latest apply of all units of `scheme` (default SFB)
        in one iteration, averaged over the live timing slots (pos_sched_timing_span)."""
        sp = C.c_float()
        _chk(lib().pos_sched_timing_span(self.h, POS_SCHEME_SFB if scheme is None else scheme,
                                         C.byref(sp)), "pos_sched_timing_span")
        return sp.value

    def close(self):
        """pos_sched_destroy. With world > 1 this frees symmetric windows (COLLECTIVE): call it
        explicitly on every rank in the same order."""
        if self.h:
            lib().pos_sched_destroy(self.h)
            self.h = None

    def __del__(self):
        if getattr(self, "h", None):
            if self.ctx.world > 1 and not self.ctx.local:
                import warnings
                warnings.warn("poseidon Scheduler (world > 1) garbage-collected without close(): leaked")
                return
            try:
                self.close()
            except Exception:
                pass


__all__ = [n for n in dir() if n.startswith(("pos_", "POS_"))] + [
    "Context", "Scheduler", "LoopFC", "PoseidonError", "DTYPES", "SCHEME_NAMES", "LIB_PATH", "lib"]
