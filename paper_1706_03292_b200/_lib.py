"""ctypes loader for libposeidon.so — argument marshalling only.

Every entry point of include/poseidon.h is declared here with the same name. There is no Python
or CPU fallback: if the shared library is missing, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os

LIB_PATH = os.environ.get("POS_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libposeidon.so")

i32, i64, u64, f32, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_void_p
P_i64, P_u64, P_f32 = C.POINTER(C.c_int64), C.POINTER(C.c_uint64), C.POINTER(C.c_float)
f64, P_f64 = C.c_double, C.POINTER(C.c_double)

# name -> (restype, argtypes); mirrors include/poseidon.h
SIGNATURES = {
    "pos_version": (C.c_int, []),
    "pos_last_error": (C.c_char_p, []),
    "pos_choose_scheme": (C.c_int, [i64, i64, i64, i32]),
    "pos_choose_scheme2": (C.c_int, [i32, i64, i64, i64, i32, i32]),
    "pos_cost_elems": (C.c_int, [i32, i32, i64, i64, i64, i32, i32, P_u64, P_u64]),
    "pos_shard_stride": (i64, [i64, i32]),
    "pos_shard_range": (C.c_int, [i64, i32, i32, P_i64, P_i64]),
    "pos_scheme_times_b200": (C.c_int, [i64, i64, i64, i32, i32, f64, f64, f64, P_f64, P_f64]),
    "pos_scheme_time_adam_b200": (C.c_int, [i64, i64, i64, i32, i32, f64, f64, f64, P_f64]),
    "pos_padded_size": (i64, [i64, i32]),
    "pos_factor_row_elems": (i64, [i64, i64]),
    "pos_factor_slot_rows": (i64, [i64, i32]),
    "pos_get_unique_id": (C.c_int, [vp]),
    "pos_init": (C.c_int, [vp, i32, i32, C.POINTER(vp)]),
    "pos_init_local": (C.c_int, [i32, C.POINTER(vp)]),
    "pos_finalize": (C.c_int, [vp]),
    "pos_world": (C.c_int, [vp]),
    "pos_rank": (C.c_int, [vp]),
    "pos_get_async_error": (C.c_int, [vp]),
    "pos_set_max_ctas": (C.c_int, [vp, i32]),
    "pos_set_timeout_ms": (C.c_int, [vp, i64]),
    "pos_set_reduce_order": (C.c_int, [vp, i32]),
    "pos_inject_fault": (C.c_int, [vp, i32, i32]),
    "pos_mem_alloc": (C.c_int, [vp, i64, C.POINTER(vp)]),
    "pos_mem_free": (C.c_int, [vp, vp]),
    "pos_mem_is_symmetric": (C.c_int, [vp, vp, i64]),
    "pos_pack_factors": (C.c_int, [i64, i64, i64, i32, i32, vp, vp, vp, vp]),
    "pos_reconstruct_apply": (C.c_int, [i64, i64, i64, i32, vp, i32, vp, i64, vp, f32, vp]),
    "pos_ps_apply": (C.c_int, [vp, vp, i64, f32, vp]),
    "pos_sync_layer_sfb": (C.c_int, [vp, i64, i64, i64, i32, i32, vp, vp, vp, vp, f32, vp]),
    "pos_sync_layer_ps": (C.c_int, [vp, i64, vp, vp, f32, vp]),
    "pos_sync_layer_fc_ps": (C.c_int, [vp, i64, i64, i64, i32, i32, vp, vp, vp, vp, i32, f32, vp]),
    "pos_sim_sync_layer_sfb": (C.c_int, [vp, i64, i64, i64, i32, i32, C.POINTER(vp), C.POINTER(vp),
                                         vp, vp, f32, vp]),
    "pos_sim_sync_layer_ps": (C.c_int, [vp, i64, C.POINTER(vp), vp, f32, vp]),
    "pos_loop_sync_layer_ps_ce": (C.c_int, [vp, i64, C.POINTER(vp), C.POINTER(vp), f32, vp]),
    "pos_loop_sync_layer_ps": (C.c_int, [vp, i64, C.POINTER(vp), C.POINTER(vp), f32, vp]),
    "pos_loop_fc_create": (C.c_int, [vp, i64, i64, i64, i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "pos_loop_fc_sync": (C.c_int, [vp, i32, C.POINTER(vp), C.POINTER(vp), f32, vp]),
    "pos_loop_fc_destroy": (C.c_int, [vp]),
    "pos_sched_create": (C.c_int, [vp, i32, i32, C.POINTER(vp)]),
    "pos_sched_add_fc": (C.c_int, [vp, i32, i64, i64, i64, i32, i32, vp, vp, vp, i32]),
    "pos_sched_add_dense": (C.c_int, [vp, i32, i64, vp, vp]),
    "pos_sched_add_dense_bucket": (C.c_int, [vp, i32, i32, P_i64, vp, vp]),
    "pos_sched_unit_of": (C.c_int, [vp, i32]),
    "pos_sched_begin": (C.c_int, [vp, f32]),
    "pos_sched_factors_ready": (C.c_int, [vp, i32, i64, vp, vp, vp, vp]),
    "pos_sched_grad_ready": (C.c_int, [vp, i32, vp]),
    "pos_sched_wait": (C.c_int, [vp, i64]),
    "pos_sched_wait_layer": (C.c_int, [vp, i32, vp]),
    "pos_sched_end": (C.c_int, [vp, vp]),
    "pos_sched_end_layers": (C.c_int, [vp, vp]),
    "pos_sched_scheme": (C.c_int, [vp, i32]),
    "pos_sched_timing": (C.c_int, [vp, i32, P_f32, P_f32, P_f32]),
    "pos_sched_timing_reset": (C.c_int, [vp]),
    "pos_sched_timeline": (C.c_int, [vp, P_f32, i32]),
    "pos_sched_trace": (C.c_int, [vp, i32, P_f64, P_f64, P_i64]),
    "pos_sched_trace_span": (C.c_int, [vp, i32, P_f64, P_i64]),
    "pos_sched_trace_last": (C.c_int, [vp, i32, P_i64, P_i64]),
    "pos_sched_trace_reset": (C.c_int, [vp]),
    "pos_sched_set_trace": (C.c_int, [vp, i32]),
    "pos_sched_timing_span": (C.c_int, [vp, i32, P_f32]),
    "pos_sched_destroy": (C.c_int, [vp]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built. Run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(nvcc, sm_100a). There is no CPU fallback.")
        h = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib
