// WFBP scheduler — wait-free backpropagation (§3.1) as Algorithm 2
// on CUDA streams and events instead of a CPU thread pool.
//
//  * one record per layer = the paper's "syncer", with its scheme fixed at
//    registration by Algorithm 1 ("choose the optimal method even before the
//    communication happens");
//  * a trigger (pos_sched_factors_ready / pos_sched_grad_ready) is Alg. 2 L7
//    "thread_pool.Schedule(sync(l))": it records an event on the producer (backward) stream and
//    enqueues the layer's sync behind that event, so s^l overlaps b^i for i < l;
//  * all collectives go on ONE high-priority comm stream in trigger order (the same L..1 order on
//    every rank — a requirement of NCCL); the heavy SFB reconstruct-and-apply runs on a pool of
//    apply streams (the paper's GPU stream pool);
//  * the binary vector C is one completion event per layer; pos_sched_end makes the
//    consumer stream wait for all of them (Alg. 2 L8 "wait_until(sync_count == num_layers)").
//  * POS_SCHED_SEQUENTIAL defers every sync until pos_sched_end, behind an event recorded on the
//    consumer stream: the "sync after the whole backward" baseline (Fig. 3a; the
//    Caffe+PS comparison of PAPER:407).
#include <vector>

#include "ctx.h"

namespace {

constexpr int kPool = 4;
constexpr int kTRing = 4;   // timing event sets per layer (iterations in flight)

struct TSlot {
  cudaEvent_t start = nullptr, packed = nullptr, gathered = nullptr, a0 = nullptr, a1 = nullptr,
              done = nullptr;
  bool used = false;
};

struct Layer {
  bool added = false;
  int kind = POS_KIND_DENSE;
  int scheme = POS_SCHEME_PS;
  int64_t M = 0, N = 0, K = 0, n = 0;
  int32_t in_dtype = POS_IN_F32, dtype = POS_DT_BF16;
  float* W = nullptr;
  float* b = nullptr;
  float* grad = nullptr;
  void* gbuf = nullptr;   // SFB: P*K rows of the gathered factors; FC-on-PS: K rows (local)
  cudaEvent_t ev_ready = nullptr, ev_gathered = nullptr, ev_done = nullptr;
  TSlot ring[kTRing];
  double acc_pack = 0, acc_comm = 0, acc_apply = 0;
  int64_t n_acc = 0;
  bool triggered = false;
  const void* u = nullptr;
  const void* v = nullptr;
  int64_t trig_seq = -1;
};

}  // namespace

struct pos_sched {
  pos_ctx* ctx = nullptr;
  int L = 0;
  int flags = 0;
  std::vector<Layer> layers;
  cudaStream_t pool[kPool] = {};
  bool in_iter = false;
  float alpha = 0.0f;
  int n_triggered = 0;
  std::vector<int> order;  // trigger order of the current iteration
  cudaEvent_t ev_end = nullptr;
  int64_t iter = 0;        // iterations begun
};

using namespace pos;

namespace {

bool timing(const pos_sched* s) { return (s->flags & POS_SCHED_TIMING) != 0; }

int make_event(cudaEvent_t* e, bool timed) {
  POS_CUDA_TRY(cudaEventCreateWithFlags(e, timed ? cudaEventDefault : cudaEventDisableTiming));
  return POS_OK;
}

// Fold a finished iteration's timing events into the layer's running sums.
int harvest(Layer& ly, TSlot& t) {
  if (!t.used) return POS_OK;
  POS_CUDA_TRY(cudaEventSynchronize(t.done));
  float pack = 0, comm = 0, apply = 0, extra = 0;
  POS_CUDA_TRY(cudaEventElapsedTime(&pack, t.start, t.packed));
  if (ly.scheme == POS_SCHEME_SFB) {
    POS_CUDA_TRY(cudaEventElapsedTime(&comm, t.packed, t.gathered));   // all-gather
    POS_CUDA_TRY(cudaEventElapsedTime(&apply, t.a0, t.a1));            // reconstruct-and-apply
  } else {
    POS_CUDA_TRY(cudaEventElapsedTime(&comm, t.packed, t.a0));         // reduce-scatter
    POS_CUDA_TRY(cudaEventElapsedTime(&apply, t.a0, t.a1));            // shard apply
    POS_CUDA_TRY(cudaEventElapsedTime(&extra, t.a1, t.done));          // all-gather
    comm += extra;
  }
  ly.acc_pack += pack;
  ly.acc_comm += comm;
  ly.acc_apply += apply;
  ly.n_acc += 1;
  t.used = false;
  return POS_OK;
}

// Enqueue sync(l) behind ly.ev_ready.
int issue_layer(pos_sched* s, int l) {
  pos_ctx* c = s->ctx;
  Layer& ly = s->layers[l];
  cudaStream_t cs = c->comm_stream;
  const bool tm = timing(s);
  const int P = c->world;
  TSlot* ts = nullptr;
  if (tm) {
    ts = &ly.ring[(s->iter - 1) % kTRing];
    int rc0 = harvest(ly, *ts);
    if (rc0) return rc0;
    ts->used = true;
  }
  POS_CUDA_TRY(cudaStreamWaitEvent(cs, ly.ev_ready, 0));
  if (s->flags & POS_SCHED_SEQUENTIAL) POS_CUDA_TRY(cudaStreamWaitEvent(cs, s->ev_end, 0));
  if (tm) POS_CUDA_TRY(cudaEventRecord(ts->start, cs));
  int rc = POS_OK;
  if (ly.scheme == POS_SCHEME_SFB) {
    const int64_t R = row_elems(ly.M, ly.N), slot = ly.K * R;
    uint8_t* my_slot =
        static_cast<uint8_t*>(ly.gbuf) + (size_t)(c->rank * slot * dtype_bytes(ly.dtype));
    // Move(GPU2CPU) analogue: A2 pack into this rank's slot
    cudaError_t e = launch_pack_factors(ly.M, ly.N, ly.K, ly.in_dtype, ly.dtype, ly.u, ly.v,
                                        my_slot, cs);
    if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack launch");
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->packed, cs));
    // Send + Receive: A3 all-gather of the factors
    if (P > 1) {
      ncclResult_t r = ncclAllGather(my_slot, ly.gbuf, (size_t)slot, nccl_type(ly.dtype), c->comm, cs);
      if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclAllGather(factors)");
    }
    POS_CUDA_TRY(cudaEventRecord(ly.ev_gathered, cs));
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->gathered, cs));
    // Move(CPU2GPU) analogue: A4 + A4b on an apply stream
    cudaStream_t as = s->pool[l % kPool];
    POS_CUDA_TRY(cudaStreamWaitEvent(as, ly.ev_gathered, 0));
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->a0, as));
    rc = reconstruct_apply(ly.M, ly.N, ly.K * P, ly.dtype, ly.gbuf, 1, ly.W, ly.N, ly.b, s->alpha,
                           c->max_ctas, as);
    if (rc != POS_OK) { if (c->sticky == POS_OK) c->sticky = rc; return rc; }
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->a1, as));
    POS_CUDA_TRY(cudaEventRecord(ly.ev_done, as));
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->done, as));
  } else {
    int64_t n = ly.n;
    if (ly.kind == POS_KIND_FC) {
      // FC layer on the PS path: local dense gradient from the factors first
      rc = stage_fc_local_grad(c, ly.M, ly.N, ly.K, ly.in_dtype, ly.dtype, ly.u, ly.v, ly.gbuf,
                               ly.grad, ly.b != nullptr, cs);
      if (rc != POS_OK) return rc;
    }
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->packed, cs));
    rc = stage_ps_dense(c, n, ly.grad, ly.W, s->alpha, cs, tm ? ts->a0 : nullptr,
                        tm ? ts->a1 : nullptr);
    if (rc != POS_OK) return rc;
    POS_CUDA_TRY(cudaEventRecord(ly.ev_done, cs));
    if (tm) POS_CUDA_TRY(cudaEventRecord(ts->done, cs));
  }
  return POS_OK;
}

int check_layer(pos_sched* s, int32_t l) {
  POS_CHECK_ARG(s, "NULL scheduler");
  POS_CHECK_ARG(l >= 0 && l < s->L, "layer %d out of [0, %d)", l, s->L);
  return POS_OK;
}

int trigger(pos_sched* s, int32_t l, cudaStream_t st) {
  Layer& ly = s->layers[l];
  if (!s->in_iter) POS_FAIL(POS_ESTATE, "trigger of layer %d outside begin/end", l);
  if (ly.triggered) POS_FAIL(POS_ESTATE, "layer %d triggered twice in one iteration", l);
  POS_CUDA_TRY(cudaEventRecord(ly.ev_ready, st));
  ly.triggered = true;
  ly.trig_seq = s->n_triggered++;
  s->order.push_back(l);
  if (s->flags & POS_SCHED_SEQUENTIAL) return POS_OK;  // deferred to pos_sched_end
  return issue_layer(s, l);
}

}  // namespace

extern "C" {

int pos_sched_create(pos_ctx* c, int32_t n_layers, int32_t flags, pos_sched** out) {
  clear_error();
  POS_CHECK_ARG(c && out, "NULL argument");
  POS_CHECK_ARG(n_layers >= 1, "n_layers must be >= 1");
  POS_CHECK_ARG((flags & ~(POS_SCHED_TIMING | POS_SCHED_SEQUENTIAL)) == 0, "unknown flags");
  POS_CHECK_ARG(!c->local || c->world == 1, "the scheduler needs a real (or 1-worker) context");
  pos_sched* s = new pos_sched();
  s->ctx = c;
  s->L = n_layers;
  s->flags = flags;
  s->layers.resize(n_layers);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  for (int i = 0; i < kPool; ++i) {
    cudaError_t e = cudaStreamCreateWithPriority(&s->pool[i], cudaStreamNonBlocking, lo);
    if (e != cudaSuccess) { pos_sched_destroy(s); return ctx_cuda_fail(c, e, "stream create"); }
  }
  if (cudaEventCreateWithFlags(&s->ev_end, cudaEventDisableTiming) != cudaSuccess) {
    pos_sched_destroy(s);
    POS_FAIL(POS_ECUDA, "event create failed");
  }
  *out = s;
  return POS_OK;
}

static int add_common(pos_sched* s, int32_t l) {
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (s->in_iter) POS_FAIL(POS_ESTATE, "add after begin");
  if (s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d added twice", l);
  Layer& ly = s->layers[l];
  const bool tm = timing(s);
  if ((rc = make_event(&ly.ev_ready, false)) || (rc = make_event(&ly.ev_gathered, false)) ||
      (rc = make_event(&ly.ev_done, false)))
    return rc;
  if (tm)
    for (auto& t : ly.ring)
      if ((rc = make_event(&t.start, true)) || (rc = make_event(&t.packed, true)) ||
          (rc = make_event(&t.gathered, true)) || (rc = make_event(&t.a0, true)) ||
          (rc = make_event(&t.a1, true)) || (rc = make_event(&t.done, true)))
        return rc;
  return POS_OK;
}

int pos_sched_add_fc(pos_sched* s, int32_t l, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                     int32_t dtype, float* W, float* b, float* grad, int32_t force_scheme) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  pos_ctx* c = s->ctx;
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && M <= (1LL << 31) && N <= (1LL << 31),
                "bad M, N, K");
  POS_CHECK_ARG(in_dtype == POS_IN_BF16 || in_dtype == POS_IN_F32, "bad in_dtype");
  POS_CHECK_ARG(dtype == POS_DT_BF16 || dtype == POS_DT_TF32 || dtype == POS_DT_F32, "bad dtype");
  POS_CHECK_ARG(W, "NULL W");
  POS_CHECK_ARG(force_scheme == -1 || force_scheme == POS_SCHEME_PS ||
                    force_scheme == POS_SCHEME_SFB,
                "bad force_scheme");
  int scheme = force_scheme >= 0 ? force_scheme : pos_choose_scheme(M, N, K, c->world);
  if (scheme < 0) return scheme;
  const int64_t n = M * N + (b ? M : 0);
  if (scheme == POS_SCHEME_PS) {
    POS_CHECK_ARG(grad, "FC layer on the PS path needs a grad buffer");
    POS_CHECK_ARG(!b || b == W + M * N, "FC layer on the PS path needs b == W + M*N");
    POS_CHECK_ARG(aligned16(W) && aligned16(grad), "W and grad must be 16-byte aligned");
  }
  if ((rc = add_common(s, l))) return rc;
  Layer& ly = s->layers[l];
  ly.kind = POS_KIND_FC;
  ly.scheme = scheme;
  ly.M = M; ly.N = N; ly.K = K; ly.n = n;
  ly.in_dtype = in_dtype; ly.dtype = dtype;
  ly.W = W; ly.b = b; ly.grad = grad;
  const int64_t rows = scheme == POS_SCHEME_SFB ? K * c->world : K;
  size_t bytes = (size_t)(rows * row_elems(M, N) * dtype_bytes(dtype));
  cudaError_t e = cudaMalloc(&ly.gbuf, bytes);
  if (e != cudaSuccess) { (void)cudaGetLastError(); POS_FAIL(POS_ENOMEM, "cudaMalloc(%zu)", bytes); }
  ly.added = true;
  return scheme;
}

int pos_sched_add_dense(pos_sched* s, int32_t l, int64_t n, float* W, float* grad) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  POS_CHECK_ARG(n >= 1, "n must be >= 1");
  POS_CHECK_ARG(W && grad && aligned16(W) && aligned16(grad), "W, grad: non-NULL, 16-byte aligned");
  if ((rc = add_common(s, l))) return rc;
  Layer& ly = s->layers[l];
  ly.kind = POS_KIND_DENSE;
  ly.scheme = POS_SCHEME_PS;
  ly.n = n;
  ly.W = W; ly.grad = grad;
  ly.added = true;
  return POS_SCHEME_PS;
}

int pos_sched_begin(pos_sched* s, float alpha) {
  clear_error();
  POS_CHECK_ARG(s, "NULL scheduler");
  if (s->in_iter) POS_FAIL(POS_ESTATE, "begin twice without end");
  for (int l = 0; l < s->L; ++l)
    if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d was never added", l);
  int rc = ctx_check(s->ctx);
  if (rc) return rc;
  for (auto& ly : s->layers) { ly.triggered = false; ly.trig_seq = -1; }  // C := 0
  s->order.clear();
  s->n_triggered = 0;
  s->alpha = alpha;
  s->in_iter = true;
  s->iter += 1;
  return POS_OK;
}

int pos_sched_factors_ready(pos_sched* s, int32_t l, const void* u, const void* v, void* stream) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  Layer& ly = s->layers[l];
  if (ly.kind != POS_KIND_FC) POS_FAIL(POS_ESTATE, "layer %d is not an FC layer", l);
  POS_CHECK_ARG(u && v, "NULL factors");
  ly.u = u;
  ly.v = v;
  return trigger(s, l, (cudaStream_t)stream);
}

int pos_sched_grad_ready(pos_sched* s, int32_t l, void* stream) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (s->layers[l].kind != POS_KIND_DENSE) POS_FAIL(POS_ESTATE, "layer %d is not a dense layer", l);
  return trigger(s, l, (cudaStream_t)stream);
}

int pos_sched_wait_layer(pos_sched* s, int32_t l, void* consumer) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!s->layers[l].triggered && s->in_iter) POS_FAIL(POS_ESTATE, "layer %d not triggered yet", l);
  POS_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)consumer, s->layers[l].ev_done, 0));
  return POS_OK;
}

int pos_sched_end(pos_sched* s, void* consumer) {
  clear_error();
  POS_CHECK_ARG(s, "NULL scheduler");
  if (!s->in_iter) POS_FAIL(POS_ESTATE, "end without begin");
  if (s->n_triggered != s->L) {
    POS_FAIL(POS_ESTATE, "end with %d of %d layers triggered", s->n_triggered, s->L);
  }
  cudaStream_t cs = (cudaStream_t)consumer;
  if (s->flags & POS_SCHED_SEQUENTIAL) {
    POS_CUDA_TRY(cudaEventRecord(s->ev_end, cs));
    for (int l : s->order) {
      int rc = issue_layer(s, l);
      if (rc) { s->in_iter = false; return rc; }
    }
  }
  for (auto& ly : s->layers) POS_CUDA_TRY(cudaStreamWaitEvent(cs, ly.ev_done, 0));
  s->in_iter = false;
  return ctx_check(s->ctx);
}

int pos_sched_scheme(pos_sched* s, int32_t l) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  return s->layers[l].scheme;
}

int pos_sched_timing(pos_sched* s, int32_t l, float* pack_ms, float* comm_ms, float* apply_ms) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!timing(s)) POS_FAIL(POS_ESTATE, "scheduler created without POS_SCHED_TIMING");
  Layer& ly = s->layers[l];
  for (auto& t : ly.ring)
    if ((rc = harvest(ly, t))) return rc;
  if (ly.n_acc == 0) POS_FAIL(POS_ESTATE, "no timed iteration of layer %d yet", l);
  if (pack_ms) *pack_ms = (float)(ly.acc_pack / ly.n_acc);
  if (comm_ms) *comm_ms = (float)(ly.acc_comm / ly.n_acc);
  if (apply_ms) *apply_ms = (float)(ly.acc_apply / ly.n_acc);
  return (int)(ly.n_acc > INT32_MAX ? INT32_MAX : ly.n_acc);
}

int pos_sched_timing_reset(pos_sched* s) {
  clear_error();
  POS_CHECK_ARG(s, "NULL scheduler");
  if (!timing(s)) POS_FAIL(POS_ESTATE, "scheduler created without POS_SCHED_TIMING");
  for (auto& ly : s->layers) {
    for (auto& t : ly.ring) {
      int rc = harvest(ly, t);
      if (rc) return rc;
    }
    ly.acc_pack = ly.acc_comm = ly.acc_apply = 0;
    ly.n_acc = 0;
  }
  return POS_OK;
}

int pos_sched_destroy(pos_sched* s) {
  clear_error();
  if (!s) return POS_OK;
  for (auto& ly : s->layers) {
    if (ly.ev_done) cudaEventSynchronize(ly.ev_done);
    cudaEvent_t evs[] = {ly.ev_ready, ly.ev_gathered, ly.ev_done};
    for (cudaEvent_t e : evs)
      if (e) cudaEventDestroy(e);
    for (auto& t : ly.ring) {
      cudaEvent_t te[] = {t.start, t.packed, t.gathered, t.a0, t.a1, t.done};
      for (cudaEvent_t e : te)
        if (e) cudaEventDestroy(e);
    }
    if (ly.gbuf) cudaFree(ly.gbuf);
  }
  for (auto st : s->pool)
    if (st) cudaStreamDestroy(st);
  if (s->ev_end) cudaEventDestroy(s->ev_end);
  delete s;
  return POS_OK;
}

}  // extern "C"
