// Context lifetime, NCCL communicator, and the one-shot per-layer synchronisation entry points
// (SURVEY §8(a) A2-A8, §8(b)). Each entry point only validates, enqueues kernels and NCCL calls
// on the caller's stream, and returns; no host synchronisation on the hot path.
#include <cstdlib>
#include <cstring>

#include "ctx.h"

namespace pos {

int ctx_cuda_fail(pos_ctx* c, cudaError_t e, const char* what) {
  if (c && c->sticky == POS_OK) c->sticky = POS_ECUDA;
  POS_FAIL(POS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

int ctx_nccl_fail(pos_ctx* c, ncclResult_t r, const char* what) {
  if (c && c->sticky == POS_OK) c->sticky = POS_ENCCL;
  POS_FAIL(POS_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

int ctx_check(pos_ctx* c) {
  if (c->sticky == POS_OK && c->err_host && *c->err_host != 0) {
    c->sticky = POS_ETIMEOUT;
    POS_FAIL(POS_ETIMEOUT, "watchdog: %s — timed out after %.3f s (rank %d of %d)",
             site_name(*c->err_host), c->timeout_ns * 1e-9, c->rank, c->world);
  }
  if (c->sticky != POS_OK) POS_FAIL(c->sticky, "context has a sticky asynchronous error");
  if (c->comm) {
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c->comm, &ar);
    if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclCommGetAsyncError");
    if (ar != ncclSuccess && ar != ncclInProgress) return ctx_nccl_fail(c, ar, "NCCL async error");
  }
  return POS_OK;
}

int ctx_workspace(pos_ctx* c, size_t bytes, void** out) {
  if (bytes > c->ws_bytes) {
    if (c->ws) {
      cudaError_t e = cudaFree(c->ws);  // implicit device sync: previous users are done
      c->ws = nullptr;
      c->ws_bytes = 0;
      if (e != cudaSuccess) return ctx_cuda_fail(c, e, "cudaFree(workspace)");
    }
    size_t want = (bytes + (1u << 20) - 1) & ~size_t((1u << 20) - 1);
    cudaError_t e = cudaMalloc(&c->ws, want);
    if (e != cudaSuccess) {
      c->ws = nullptr;
      (void)cudaGetLastError();
      POS_FAIL(POS_ENOMEM, "cudaMalloc(%zu) for workspace: %s", want, cudaGetErrorString(e));
    }
    c->ws_bytes = want;
  }
  *out = c->ws;
  return POS_OK;
}

// A5 + A6 + A7 + A8 for a dense (or flattened FC) layer of n parameters, on stream s.
int ps_stage_grid(pos_ctx* c, int64_t n, float* grad, float* W, void* ce_buf) {
  const int P = c->world;
  if (P > 1 && !c->local) {
    const int64_t padded = pos_padded_size(n, P);
    if (ce_buf && symm_lookup(c, W, (size_t)padded * 4) &&
        symm_lookup(c, ce_buf, (size_t)symm_ce_bytes(n, P)))
      return symm_ce_grid(c, n);
    if (symm_lookup(c, grad, (size_t)padded * 4) && symm_lookup(c, W, (size_t)padded * 4))
      return symm_ps_grid(c, n);
  }
  int64_t lo = 0, hi = n;
  if (!c->local) pos_shard_range(n, P, c->rank, &lo, &hi);
  return hi > lo ? ps_apply_grid(hi - lo) : 0;
}

int stage_ps_dense(pos_ctx* c, int64_t n, float* grad, float* W, float alpha, cudaStream_t s,
                   cudaEvent_t ev_rs_done, cudaEvent_t ev_apply_done, bool zero_tail, KTrace tr,
                   KTrace tg, int lane, void* ce_buf, uint32_t* exit_word, bool* deferred) {
  if (deferred) *deferred = false;
  const int P = c->world;
  const int64_t S = pos_shard_stride(n, P);
  if (S < 0) return (int)S;
  if (ce_buf) {  // copy-engine transport (POS_PS_CE)
    bool done = false;
    int rc = symm_ps_ce(c, n, grad, W, ce_buf, alpha, s, ev_rs_done, ev_apply_done, &done, tr, tg);
    if (rc != POS_OK || done) return rc;
  }
  {  // NVLS fused kernel when grad and W live in symmetric memory (NEXT-1)
    bool done = false;
    int rc = symm_ps_fused(c, n, grad, W, alpha, s, ev_rs_done, ev_apply_done, &done, tr, tg, lane,
                           exit_word);
    if (deferred) *deferred = done && exit_word != nullptr;
    if (rc != POS_OK || done) return rc;
  }
  const int64_t padded = S * P;
  // A5: the padding tail is owned (zeroed) by the library so the reduce-scatter sums zeros there
  // (with a single worker nothing reads it)
  if (zero_tail && P > 1 && !c->local && padded > n) {
    cudaError_t e = cudaMemsetAsync(grad + n, 0, (size_t)(padded - n) * sizeof(float), s);
    if (e != cudaSuccess) return ctx_cuda_fail(c, e, "cudaMemsetAsync(grad tail)");
  }
  const int r = c->rank;
  if (P > 1 && !c->local) {
    // A6: in-place reduce-scatter (sum) -> rank r holds sum_p g_p on [rS, (r+1)S)
    ncclResult_t nr = ncclReduceScatter(grad, grad + (int64_t)r * S, (size_t)S, ncclFloat32,
                                        ncclSum, c->comm, s);
    if (nr != ncclSuccess) return ctx_nccl_fail(c, nr, "ncclReduceScatter");
  }
  if (ev_rs_done) POS_CUDA_TRY(record_timing_event(ev_rs_done, s));
  // A7: apply on the owned shard
  int64_t lo = 0, hi = n;
  if (!c->local) {
    pos_shard_range(n, P, r, &lo, &hi);
  }
  if (hi > lo) {
    cudaError_t e = launch_ps_apply(grad + lo, W + lo, hi - lo, alpha, s, tr, tg);
    if (e != cudaSuccess) return ctx_cuda_fail(c, e, "ps_apply launch");
  }
  if (ev_apply_done) POS_CUDA_TRY(record_timing_event(ev_apply_done, s));
  if (P > 1 && !c->local) {
    // A8: in-place all-gather of the fresh shards
    ncclResult_t nr = ncclAllGather(W + (int64_t)r * S, W, (size_t)S, ncclFloat32, c->comm, s);
    if (nr != ncclSuccess) return ctx_nccl_fail(c, nr, "ncclAllGather(W)");
  }
  return POS_OK;
}

// Local dense gradient of an FC layer on the PS path: pack this rank's K factor rows, then the
// reconstruction kernel in overwrite mode (alpha = 1): grad[0:MN] = U_r^T V_r, grad[MN:MN+M] =
// colsum(U_r).
int stage_fc_local_grad(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                        int32_t dtype, const void* u, const void* v, void* pack_buf, float* grad,
                        int32_t has_bias, cudaStream_t s) {
  cudaError_t e = launch_pack_factors(M, N, K, in_dtype, dtype, u, v, pack_buf, s);
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack launch");
  int rc = reconstruct_apply(M, N, K, dtype, pack_buf, 0, grad, N, has_bias ? grad + M * N : nullptr,
                             1.0f, c->max_ctas, s);
  if (rc != POS_OK && c->sticky == POS_OK) c->sticky = rc;
  return rc;
}

static int check_fc_args(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                         int32_t dtype) {
  POS_CHECK_ARG(c, "NULL context");
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1, "M, N, K must be >= 1");
  POS_CHECK_ARG(M <= (1LL << 31) && N <= (1LL << 31) && K <= (1LL << 31), "M, N, K too large");
  POS_CHECK_ARG(in_dtype == POS_IN_BF16 || in_dtype == POS_IN_F32, "bad in_dtype %d", in_dtype);
  POS_CHECK_ARG(dtype == POS_DT_BF16 || dtype == POS_DT_TF32 || dtype == POS_DT_F32,
                "bad dtype %d", dtype);
  return POS_OK;
}

}  // namespace pos

using namespace pos;

extern "C" {

int pos_get_unique_id(void* out_128B) {
  clear_error();
  POS_CHECK_ARG(out_128B, "NULL output");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return ctx_nccl_fail(nullptr, r, "ncclGetUniqueId");
  memcpy(out_128B, &id, sizeof(id));
  return POS_OK;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

static int ctx_common_init(pos_ctx* c) {
  POS_CUDA_TRY(cudaGetDevice(&c->device));
  // load every kernel now (lazy loading could otherwise synchronise the context at a first launch
  // while a spin-waiting kernel of this rank waits for a peer; see common.h)
  {
    static const cudaError_t preload = [] {
      cudaError_t e = preload_mem_kernels();
      if (e == cudaSuccess) e = preload_sfb_kernels();
      if (e == cudaSuccess) e = preload_symm_kernels();
      return e;
    }();
    POS_CUDA_TRY(preload);
  }
  int lo = 0, hi = 0;
  POS_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // comm stream priority: the greatest by default; POS_COMM_PRIO=n sets lo + n (clamped), an
  // experiment knob for the order in which pending PS / pack CTAs get SMs
  int prio = hi;
  if (const char* e = getenv("POS_COMM_PRIO")) prio = std::max(hi, std::min(lo, lo - atoi(e)));
  POS_CUDA_TRY(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, prio));
  c->lane_stream[0] = c->comm_stream;
  // POS_PS_LANES = 1 / 2 forces the lane count; unset (0): each scheduler decides (pos_sched_begin)
  c->ps_lanes = (int)std::max<int64_t>(0, std::min<int64_t>(kMaxLanes, env_int("POS_PS_LANES", 0)));
  POS_CUDA_TRY(cudaStreamCreateWithPriority(&c->lane_stream[1], cudaStreamNonBlocking, prio));
  // watchdog error word: host-mapped, so the host reads it without synchronising
  int* h = nullptr;
  POS_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&h), sizeof(int), cudaHostAllocMapped));
  *h = 0;
  c->err_host = h;
  POS_CUDA_TRY(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err_dev), h, 0));
  // POS_REDUCE_ORDER=0|1|2: the context's default PS reduce order (pos_set_reduce_order)
  {
    const int64_t o = env_int("POS_REDUCE_ORDER", POS_REDUCE_AUTO);
    if (o == POS_REDUCE_SWITCH || o == POS_REDUCE_RANK_ORDER || o == POS_REDUCE_AUTO) c->reduce_order = (int)o;
  }
  c->ps_ce = env_int("POS_PS_CE", 0) != 0 ? 1 : 0;
  const int64_t ms = env_int("POS_TIMEOUT_MS", 20000);
  c->timeout_ns = ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
  return POS_OK;
}

int pos_init(const void* uid, int32_t world, int32_t rank, pos_ctx** out) {
  clear_error();
  POS_CHECK_ARG(out, "NULL output");
  POS_CHECK_ARG(world >= 1 && rank >= 0 && rank < world, "bad world/rank %d/%d", world, rank);
  POS_CHECK_ARG(world == 1 || uid, "NULL unique id");
  pos_ctx* c = new pos_ctx();
  c->world = world;
  c->rank = rank;
  int rc = ctx_common_init(c);
  if (rc != POS_OK) { delete c; return rc; }
  if (world > 1) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    // NCCL's CTAs must find free SMs while the persistent reconstruction kernel runs: cap them
    // (maxCTAs) and keep the same number of SMs out of the reconstruction grid (max_ctas).
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    const int nccl_ctas = env_int("POS_NCCL_MAX_CTAS", 16);
    cfg.maxCTAs = nccl_ctas;
    cfg.commName = "poseidon";
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, world, id, rank, &cfg);
    if (r != ncclSuccess) {
      cudaStreamDestroy(c->comm_stream);
      delete c;
      return ctx_nccl_fail(nullptr, r, "ncclCommInitRankConfig");
    }
    c->max_ctas = env_int("POS_SFB_MAX_CTAS", num_sms() - nccl_ctas - 4);
  }
  *out = c;
  return POS_OK;
}

int pos_init_local(int32_t P_sim, pos_ctx** out) {
  clear_error();
  POS_CHECK_ARG(out, "NULL output");
  POS_CHECK_ARG(P_sim >= 1 && P_sim <= kMaxSimP, "P_sim must be in [1, %d]", kMaxSimP);
  pos_ctx* c = new pos_ctx();
  c->world = P_sim;
  c->rank = 0;
  c->local = true;
  int rc = ctx_common_init(c);
  if (rc != POS_OK) { delete c; return rc; }
  *out = c;
  return POS_OK;
}

int pos_finalize(pos_ctx* c) {
  clear_error();
  if (!c) return POS_OK;
  int rc = POS_OK;
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->lane_stream[1]) cudaStreamSynchronize(c->lane_stream[1]);
  symm_destroy(c);
  if (c->comm) {
    ncclResult_t r = ncclCommDestroy(c->comm);
    if (r != ncclSuccess) rc = POS_ENCCL;
  }
  if (c->ws) cudaFree(c->ws);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->lane_stream[1]) cudaStreamDestroy(c->lane_stream[1]);
  if (c->err_host) cudaFreeHost(const_cast<int*>(c->err_host));
  delete c;
  return rc;
}

int pos_world(const pos_ctx* c) { return c ? c->world : POS_EINVAL; }
int pos_rank(const pos_ctx* c) { return c ? c->rank : POS_EINVAL; }

int pos_get_async_error(pos_ctx* c) {
  clear_error();
  POS_CHECK_ARG(c, "NULL context");
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "asynchronous CUDA error");
  return ctx_check(c);
}

int pos_set_timeout_ms(pos_ctx* c, int64_t ms) {
  clear_error();
  POS_CHECK_ARG(c && ms >= 0, "bad arguments");
  c->timeout_ns = (unsigned long long)ms * 1000000ull;
  return POS_OK;
}

int pos_set_reduce_order(pos_ctx* c, int32_t order) {
  clear_error();
  POS_CHECK_ARG(c && (order == POS_REDUCE_SWITCH || order == POS_REDUCE_RANK_ORDER ||
                      order == POS_REDUCE_AUTO),
                "bad arguments");
  c->reduce_order = order;
  return POS_OK;
}

int pos_inject_fault(pos_ctx* c, int32_t kind, int32_t rank) {
  clear_error();
  POS_CHECK_ARG(c && kind >= POS_FAULT_NONE && kind <= POS_FAULT_SKIP_PACK, "bad arguments");
  c->fault = kind;
  c->fault_rank = rank;
  return POS_OK;
}

int pos_set_max_ctas(pos_ctx* c, int32_t max_ctas) {
  clear_error();
  POS_CHECK_ARG(c && max_ctas >= 0, "bad arguments");
  c->max_ctas = max_ctas;
  return POS_OK;
}

// ---------------------------------------------------------------------------- SFB one-shot --
int pos_sync_layer_sfb(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                       int32_t dtype, const void* u, const void* v, float* W, float* b,
                       float alpha, void* stream) {
  clear_error();
  int rc = check_fc_args(c, M, N, K, in_dtype, dtype);
  if (rc) return rc;
  POS_CHECK_ARG(u && v && W, "NULL pointer");
  POS_CHECK_ARG(!c->local || c->world == 1,
                "simulated context with P > 1: use pos_sim_sync_layer_sfb");
  if ((rc = ctx_check(c))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int P = c->world;
  const int64_t R = row_elems(M, N), slot = K * rows_per_sample(dtype) * R;
  void* G = nullptr;
  if ((rc = ctx_workspace(c, (size_t)(slot * P * dtype_bytes(dtype)), &G))) return rc;
  uint8_t* my_slot = static_cast<uint8_t*>(G) + (size_t)(c->rank * slot * dtype_bytes(dtype));
  // A2: pack this rank's factors into its slot of the gather buffer
  cudaError_t e = launch_pack_factors(M, N, K, in_dtype, dtype, u, v, my_slot, s);
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack launch");
  // A3: in-place all-gather of the factor blocks (P2P broadcast of SFs)
  if (P > 1) {
    ncclResult_t r = ncclAllGather(my_slot, G, (size_t)slot, nccl_type(dtype), c->comm, s);
    if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclAllGather(factors)");
  }
  // A4 + A4b
  rc = reconstruct_apply(M, N, K * P, dtype, G, 1, W, N, b, alpha, c->max_ctas, s);
  if (rc != POS_OK && c->sticky == POS_OK) c->sticky = rc;
  return rc;
}

// ----------------------------------------------------------------------------- PS one-shot --
int pos_sync_layer_ps(pos_ctx* c, int64_t n, float* grad, float* W, float alpha, void* stream) {
  clear_error();
  POS_CHECK_ARG(c, "NULL context");
  POS_CHECK_ARG(n >= 1, "n must be >= 1");
  POS_CHECK_ARG(grad && W, "NULL pointer");
  POS_CHECK_ARG(aligned16(grad) && aligned16(W), "grad and W must be 16-byte aligned");
  POS_CHECK_ARG(!c->local || c->world == 1,
                "simulated context with P > 1: use pos_sim_sync_layer_ps");
  int rc = ctx_check(c);
  if (rc) return rc;
  return stage_ps_dense(c, n, grad, W, alpha, (cudaStream_t)stream, nullptr, nullptr, true);
}

int pos_sync_layer_fc_ps(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                         int32_t dtype, const void* u, const void* v, float* grad, float* Wb,
                         int32_t has_bias, float alpha, void* stream) {
  clear_error();
  int rc = check_fc_args(c, M, N, K, in_dtype, dtype);
  if (rc) return rc;
  POS_CHECK_ARG(u && v && grad && Wb, "NULL pointer");
  POS_CHECK_ARG(aligned16(grad) && aligned16(Wb), "grad and Wb must be 16-byte aligned");
  POS_CHECK_ARG(!c->local || c->world == 1, "simulated context with P > 1 is not supported here");
  if ((rc = ctx_check(c))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  void* buf = nullptr;
  if ((rc = ctx_workspace(c, (size_t)(K * rows_per_sample(dtype) * row_elems(M, N) * dtype_bytes(dtype)),
                         &buf)))
    return rc;
  if ((rc = stage_fc_local_grad(c, M, N, K, in_dtype, dtype, u, v, buf, grad, has_bias, s)))
    return rc;
  return stage_ps_dense(c, M * N + (has_bias ? M : 0), grad, Wb, alpha, s, nullptr, nullptr,
                        true);
}

// ---------------------------------------------------------------------- simulated workers --
int pos_sim_sync_layer_sfb(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                           int32_t dtype, const void* const* u, const void* const* v, float* W,
                           float* b, float alpha, void* stream) {
  clear_error();
  int rc = check_fc_args(c, M, N, K, in_dtype, dtype);
  if (rc) return rc;
  POS_CHECK_ARG(c->local, "pos_sim_* needs a context from pos_init_local");
  POS_CHECK_ARG(u && v && W, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  const int P = c->world;
  const int64_t slot = K * rows_per_sample(dtype) * row_elems(M, N);
  void* G = nullptr;
  if ((rc = ctx_workspace(c, (size_t)(slot * P * dtype_bytes(dtype)), &G))) return rc;
  for (int p = 0; p < P; ++p) {
    POS_CHECK_ARG(u[p] && v[p], "NULL factor pointer for worker %d", p);
    uint8_t* dst = static_cast<uint8_t*>(G) + (size_t)(p * slot * dtype_bytes(dtype));
    cudaError_t e = launch_pack_factors(M, N, K, in_dtype, dtype, u[p], v[p], dst, s);
    if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack launch");
  }
  rc = reconstruct_apply(M, N, K * P, dtype, G, 1, W, N, b, alpha, c->max_ctas, s);
  if (rc != POS_OK && c->sticky == POS_OK) c->sticky = rc;
  return rc;
}

int pos_sim_sync_layer_ps(pos_ctx* c, int64_t n, const float* const* grads, float* W, float alpha,
                          void* stream) {
  clear_error();
  POS_CHECK_ARG(c && c->local, "pos_sim_* needs a context from pos_init_local");
  POS_CHECK_ARG(n >= 1 && grads && W, "bad arguments");
  for (int p = 0; p < c->world; ++p) POS_CHECK_ARG(grads[p], "NULL gradient for worker %d", p);
  cudaError_t e = launch_sim_ps_reduce_apply(grads, c->world, W, n, alpha, (cudaStream_t)stream);
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "sim reduce-apply launch");
  return POS_OK;
}

}  // extern "C"
