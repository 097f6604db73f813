// WFBP scheduler — wait-free backpropagation (§3.1) as Algorithm 2
// on CUDA streams and events instead of a CPU thread pool.
//
//  * one "syncer" per layer; its scheme is fixed at registration by Algorithm 1
//    ("choose the optimal method even before the communication happens");
//  * the synchronisation UNIT is a layer, or a BUCKET of consecutive dense layers laid out in one
//    flat buffer — the paper's fixed-size KV pairs (PAPER:258, 2 MB) as the unit of PS traffic.
//    A bucket is synchronised once all of its layers have been triggered;
//  * a trigger (pos_sched_factors_ready / pos_sched_grad_ready) is Alg. 2 L7
//    "thread_pool.Schedule(sync(l))": it records an event on the producer (backward) stream and
//    enqueues the unit's sync behind it, so s^l overlaps b^i for i < l;
//  * with collectives (P > 1) every NCCL call goes on ONE high-priority comm stream in trigger
//    order (the same L..1 order on every rank, as NCCL requires); the heavy SFB
//    reconstruct-and-apply runs on an apply stream. Without collectives (P = 1) there is no comm
//    hop: SFB units run on apply stream 0 and dense units spread over apply streams 1..3 (the
//    paper's GPU stream pool);
//  * the binary vector C is one completion event per unit; pos_sched_end makes the
//    consumer stream wait for all of them (Alg. 2 L8 "wait_until(sync_count == num_layers)");
//  * POS_SCHED_SEQUENTIAL defers every sync until pos_sched_end, behind an event recorded on the
//    consumer stream: the "sync after the whole backward" baseline (Fig. 3a; the
//    Caffe+PS comparison of PAPER:407);
//  * iterations may be captured into CUDA graphs: nothing here synchronises with the host while
//    a stream is capturing, and timing events become external event nodes.
#include <chrono>
#include <cstdlib>
#include <thread>
#include <vector>

#include "ctx.h"

namespace {

constexpr int kPool = 8;    // apply streams: [0], [4], [6] reconstructions; [1..3] dense applies;
                             // [5] flag-mode factor packs (high priority); [7] completion of
                             // the PS units with a deferred exit barrier (high priority)
constexpr int kTRing = 4;   // timing event sets per unit (iterations in flight)

struct TSlot {
  cudaEvent_t start = nullptr, packed = nullptr, gathered = nullptr, a0 = nullptr, a1 = nullptr,
              done = nullptr;
  bool used = false;
};

// A synchronisation unit: one FC layer, one dense layer, or a bucket of dense layers.
struct Unit {
  int kind = POS_KIND_DENSE;
  int scheme = POS_SCHEME_PS;
  int64_t M = 0, N = 0, K = 0, n = 0;
  int32_t in_dtype = POS_IN_F32, dtype = POS_DT_BF16;
  float* W = nullptr;
  float* b = nullptr;
  float* grad = nullptr;
  void* gbuf = nullptr;        // SFB: P*K gathered factor rows; FC-on-PS: K local rows
  bool gbuf_symm = false;      // gbuf from pos_mem_alloc (NVLS multicast target)
  // flag-mode gather (symmetric, tensor-core path): gbuf2 = second buffer, gflags = P ready
  // flags, all in gbuf's allocation; gstate = this rank's gather sequence + pack CTA counter
  bool flag_mode = false;
  void* gbuf2 = nullptr;
  uint32_t* gflags = nullptr;
  unsigned* gstate = nullptr;
  void* ce_buf = nullptr;      // PS over the copy engines (ctx->ps_ce): receive slots + flags
  uint32_t* exit_word = nullptr;   // fused PS kernel with a deferred exit: its epoch (device)
  cudaEvent_t ev_issued = nullptr; // ... recorded after its launch; the exit wait follows it
  pos::SfbTcPlan plan;         // cached TMA descriptors of the tensor-core reconstruction
  bool has_plan = false;
  int plan_ctas = -1;
  unsigned int* tile_counter = nullptr;   // dynamic tile scheduler state of this unit's launches
  unsigned long long* trace = nullptr;    // POS_SCHED_TRACE: device-side record of the apply kernel
  int trace_grid = 0;                     // CTAs of one traced launch (0 = nothing traced)
  std::vector<int> members;    // layer indices (forward order)
  int pending = 0;             // members not yet triggered in this iteration
  const void* u = nullptr;     // FC factors of this iteration
  const void* v = nullptr;
  cudaEvent_t ev_gathered = nullptr, ev_done = nullptr;
  TSlot ring[kTRing];
  double acc_pack = 0, acc_comm = 0, acc_apply = 0;
  int64_t n_acc = 0;
  int seq = 0;                 // registration order (stream assignment)
  int sfb_idx = 0;             // index among the SFB units (reconstruction stream assignment)
};

struct Layer {
  bool added = false;
  int kind = POS_KIND_DENSE;
  int unit = -1;
  bool triggered = false;
  // the caller's events of this iteration's trigger: inputs ready (factors / gradient) and, for
  // an FC layer, W no longer read by b^l (nullptr = same as ev_in)
  cudaEvent_t ev_in = nullptr, ev_wfree = nullptr;
};

}  // namespace

struct pos_sched {
  pos_ctx* ctx = nullptr;
  int L = 0;
  int flags = 0;
  std::vector<Layer> layers;
  std::vector<Unit> units;
  cudaStream_t pool[kPool] = {};
  bool in_iter = false;
  float alpha = 0.0f;
  int n_triggered = 0;
  std::vector<int> order;  // unit issue order of the current iteration
  cudaEvent_t ev_end = nullptr;
  int64_t iter = 0;        // iterations begun
  bool captured = false;   // some iteration was issued under CUDA-graph stream capture
  int last_sfb = -1;       // most recently issued SFB unit of this iteration
  bool ps_after_sfb = false;  // P > 1: dense units wait for the SFB reconstructions (no overlap)
  int sfb_streams = 2;        // reconstruction streams (POS_SFB_STREAMS=1|2|3)
  // flag-mode packs on their own stream instead of the comm stream: the PS chain then starts with
  // the first dense unit, but the packs (and so the reconstructions) wait behind PS traffic —
  // decided per step mix at the first begin (pos_sched_begin), or forced by POS_PACK_STREAM
  int pack_stream = -1;     // flag-mode packs on pool[5]: 1 / 0 forced (POS_PACK_STREAM), -1 auto
  int lanes = 0;           // PS lanes in use (decided at the first begin unless the context forces it)
  bool defer_exit = true;   // POS_PS_DEFER=0: the fused PS kernels wait at their exit barrier
  int n_sfb = 0;              // SFB units registered
  bool any_pair = false;      // some SFB unit reconstructs with the CTA-pair kernel
  // POS_SCHED_TRACE: one group record per scheme (all of a step's PS / SFB apply kernels)
  unsigned long long* group[2] = {nullptr, nullptr};
  unsigned group_expected[2] = {0, 0};
  int traced_ctas = -2;       // max_ctas the traced grids were computed for
};

using namespace pos;

namespace {

bool timing_full(const pos_sched* s) { return (s->flags & POS_SCHED_TIMING) != 0; }
bool tracing(const pos_sched* s) { return (s->flags & POS_SCHED_TRACE) != 0; }

// (re)build the cached tensor-core launch plan of an SFB unit for the context's current CTA cap
int ensure_plan(pos_sched* s, Unit& un) {
  pos_ctx* c = s->ctx;
  if (un.scheme != POS_SCHEME_SFB || un.plan_ctas == c->max_ctas) return POS_OK;
  un.has_plan = sfb_tc_make_plan(&un.plan, un.M, un.N, un.K * c->world, un.dtype, un.gbuf, un.W,
                                 un.N, c->max_ctas, un.b, un.flag_mode ? un.gbuf2 : nullptr,
                                 /*cluster_ok=*/c->world == 1);
  un.plan.counter = (s->flags & POS_SCHED_STATIC_TILES) ? nullptr : un.tile_counter;
  un.plan.gsel = un.flag_mode ? un.gstate : nullptr;
  if (un.flag_mode && !un.has_plan) POS_FAIL(POS_ESTATE, "flag-mode gather without a tensor-core plan");
  un.plan_ctas = c->max_ctas;
  return POS_OK;
}

// Device-side tracing: every unit's apply kernel stamps its own record; the apply kernels of one
// step also stamp the group record of their scheme, whose interval is the sum of their grids.
int prepare_tracing(pos_sched* s) {
  pos_ctx* c = s->ctx;
  if (s->traced_ctas == c->max_ctas) return POS_OK;
  unsigned exp[2] = {0, 0};
  bool complete[2] = {true, true};
  for (auto& un : s->units) {
    int rc = ensure_plan(s, un);
    if (rc) return rc;
    if (!un.trace) POS_CUDA_TRY(ktrace_alloc(&un.trace));
    const int sc = un.scheme == POS_SCHEME_SFB ? 1 : 0;
    if (un.scheme == POS_SCHEME_SFB)
      un.trace_grid = un.has_plan ? un.plan.grid : 0;        // the SIMT path is not traced
    else
      un.trace_grid = ps_stage_grid(c, un.n, un.grad, un.W, un.ce_buf);
    if (un.trace_grid > 0) exp[sc] += (unsigned)un.trace_grid;
    else if (un.scheme == POS_SCHEME_SFB) complete[sc] = false;
  }
  for (int k = 0; k < 2; ++k) {
    if (!s->group[k]) POS_CUDA_TRY(ktrace_alloc(&s->group[k]));
    POS_CUDA_TRY(ktrace_reset(s->group[k]));
    s->group_expected[k] = complete[k] ? exp[k] : 0;
  }
  for (auto& un : s->units) POS_CUDA_TRY(ktrace_reset(un.trace));
  s->traced_ctas = c->max_ctas;
  return POS_OK;
}

KTrace unit_trace(const pos_sched* s, const Unit& un) {
  KTrace t;
  if (tracing(s) && un.trace && un.trace_grid > 0) {
    t.rec = un.trace;
    t.expected = (unsigned)un.trace_grid;
  }
  return t;
}

KTrace group_trace(const pos_sched* s, int scheme) {
  KTrace t;
  const int k = scheme == POS_SCHEME_SFB ? 1 : 0;
  if (tracing(s) && s->group[k] && s->group_expected[k] > 0) {
    t.rec = s->group[k];
    t.expected = s->group_expected[k];
  }
  return t;
}
bool timing_any(const pos_sched* s) {
  return (s->flags & (POS_SCHED_TIMING | POS_SCHED_TIMING_APPLY)) != 0;
}

int make_event(cudaEvent_t* e, bool timed) {
  POS_CUDA_TRY(cudaEventCreateWithFlags(e, timed ? cudaEventDefault : cudaEventDisableTiming));
  return POS_OK;
}

int trec(cudaEvent_t e, cudaStream_t st) {
  if (!e) return POS_OK;
  POS_CUDA_TRY(record_timing_event(e, st));
  return POS_OK;
}

bool is_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive;
}

// Fold a finished iteration's timing events into the unit's running sums. Under graph replay the
// slot's events are re-recorded by every replay of the graph that owns them, so the slot stays
// `used` (keep_used) and each harvest samples the latest replay.
int harvest(Unit& u, TSlot& t, bool keep_used = false) {
  if (!t.used) return POS_OK;
  POS_CUDA_TRY(cudaEventSynchronize(t.a1));
  float pack = 0, comm = 0, apply = 0, extra = 0;
  POS_CUDA_TRY(cudaEventElapsedTime(&apply, t.a0, t.a1));
  if (t.start) {
    POS_CUDA_TRY(cudaEventSynchronize(t.done));
    POS_CUDA_TRY(cudaEventElapsedTime(&pack, t.start, t.packed));
    if (u.scheme == POS_SCHEME_SFB) {
      POS_CUDA_TRY(cudaEventElapsedTime(&comm, t.packed, t.gathered));   // all-gather
    } else {
      POS_CUDA_TRY(cudaEventElapsedTime(&comm, t.packed, t.a0));         // reduce-scatter
      POS_CUDA_TRY(cudaEventElapsedTime(&extra, t.a1, t.done));          // all-gather
      comm += extra;
    }
  }
  u.acc_pack += pack;
  u.acc_comm += comm;
  u.acc_apply += apply;
  u.n_acc += 1;
  t.used = keep_used;
  return POS_OK;
}

// Enqueue sync(unit) behind the ready events of all its member layers.
int issue_unit(pos_sched* s, int ui) {
  pos_ctx* c = s->ctx;
  Unit& un = s->units[ui];
  const int P = c->world;
  const bool coll = P > 1;                 // collectives needed?
  TSlot* ts = nullptr;
  int rc = POS_OK;
  // stream of the first stage: the comm stream when a collective follows, else an apply stream
  // Consecutive SFB reconstructions alternate between two streams: they touch different layers, so
  // the next one's CTAs can take each SM as the previous one's persistent CTAs leave (no
  // full-drain gap between them); dense applies rotate over three more streams.
  // Not with the CTA-pair (cluster) kernel: a cluster launch pending behind a running persistent
  // kernel on another stream can hold SMs that the cross-GPU kernels need (observed deadlock at
  // P = 4, AlexNet K*P = 512), so then all reconstructions stay on one stream.
  static constexpr int kSfbPool[3] = {0, 4, 6};
  const int nrs = s->any_pair ? 1 : s->sfb_streams;
  cudaStream_t as = un.scheme == POS_SCHEME_SFB ? s->pool[kSfbPool[un.sfb_idx % nrs]]
                                                : s->pool[1 + un.seq % 3];
  // first stage: the comm stream when a collective follows; else an auxiliary apply stream, so the
  // factor pack of the next SFB layer overlaps the reconstruction of this one
  cudaStream_t cs = coll ? c->comm_stream : s->pool[1 + un.seq % 3];
  // Flag-mode packs (multicast stores + ready flags, no cross-GPU barrier) need no ordering with
  // the fused PS kernels, which keep the comm stream to themselves: the PS chain then starts
  // with the first dense unit instead of queueing behind every factor pack of the step
  if (coll && un.scheme == POS_SCHEME_SFB && un.flag_mode && s->pack_stream == 1) cs = s->pool[5];
  // PS units alternate between the context's lanes by registration order (identical on every rank)
  const int lane = (coll && un.scheme != POS_SCHEME_SFB && s->lanes > 1) ? un.seq % s->lanes : 0;
  if (lane > 0) cs = c->lane_stream[lane];
  for (int l : un.members) POS_CUDA_TRY(cudaStreamWaitEvent(cs, s->layers[l].ev_in, 0));
  // the stage that WRITES W waits for b^l to have finished reading it (WAR)
  const Layer& l0 = s->layers[un.members[0]];
  cudaEvent_t ev_wfree = l0.ev_wfree ? l0.ev_wfree : l0.ev_in;
  // Optionally keep the NVLink-latency-bound PS kernels from co-running with the HBM-bound
  // reconstructions (they starve each other's memory pipelines); see DESIGN.md.
  if (coll && s->ps_after_sfb && un.scheme != POS_SCHEME_SFB && s->last_sfb >= 0)
    POS_CUDA_TRY(cudaStreamWaitEvent(cs, s->units[s->last_sfb].ev_done, 0));
  if (un.scheme == POS_SCHEME_SFB) s->last_sfb = ui;
  if (s->flags & POS_SCHED_SEQUENTIAL) POS_CUDA_TRY(cudaStreamWaitEvent(cs, s->ev_end, 0));
  // cs has joined the caller's stream capture (if any) through the waits above; inside a capture
  // nothing may synchronise with the host, so the timing slot is not harvested there
  const bool capturing = is_capturing(cs);
  s->captured |= capturing;
  if (timing_any(s)) {
    ts = &un.ring[(s->iter - 1) % kTRing];
    if (!capturing && (rc = harvest(un, *ts))) return rc;
    ts->used = true;
  }
  if (ts && (rc = trec(ts->start, cs))) return rc;
  if (un.scheme == POS_SCHEME_SFB) {
    const int64_t R = row_elems(un.M, un.N), slot = un.K * rows_per_sample(un.dtype) * R;
    uint8_t* my_slot =
        static_cast<uint8_t*>(un.gbuf) + (size_t)(c->rank * slot * dtype_bytes(un.dtype));
    // Move(GPU2CPU) + Send + Receive, fused over NVLS when the gather buffer is symmetric
    bool mc = false;
    if (coll && (rc = symm_pack_mc(c, un.M, un.N, un.K, un.in_dtype, un.dtype, un.u, un.v, un.gbuf,
                                   cs, &mc, un.flag_mode ? un.gbuf2 : nullptr, un.gflags,
                                   un.gstate)))
      return rc;
    if (un.flag_mode && !mc) POS_FAIL(POS_ESTATE, "flag-mode gather could not be launched");
    if (!mc) {
      // A2 pack into this rank's slot
      cudaError_t e = launch_pack_factors(un.M, un.N, un.K, un.in_dtype, un.dtype, un.u, un.v,
                                          my_slot, cs);
      if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack launch");
    }
    if (ts && (rc = trec(ts->packed, cs))) return rc;
    if (coll && mc && un.flag_mode) {
      // our slot is pushed; the apply stream waits for every rank's ready flag (no barrier on
      // the comm stream, which moves on to the next unit at once)
      POS_CUDA_TRY(cudaEventRecord(un.ev_gathered, cs));
      POS_CUDA_TRY(cudaStreamWaitEvent(as, un.ev_gathered, 0));
      if ((rc = symm_wait_gathered(c, un.gflags, un.gstate, P, as))) return rc;
      if (ts && (rc = trec(ts->gathered, as))) return rc;
    } else if (coll && mc) {
      if (ts && (rc = trec(ts->gathered, cs))) return rc;
      POS_CUDA_TRY(cudaEventRecord(un.ev_gathered, cs));
      POS_CUDA_TRY(cudaStreamWaitEvent(as, un.ev_gathered, 0));
    } else if (coll) {
      // Send + Receive: A3 all-gather of the factors
      ncclResult_t r =
          ncclAllGather(my_slot, un.gbuf, (size_t)slot, nccl_type(un.dtype), c->comm, cs);
      if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclAllGather(factors)");
      if (ts && (rc = trec(ts->gathered, cs))) return rc;
      POS_CUDA_TRY(cudaEventRecord(un.ev_gathered, cs));   // sync events last: joins a capture
      POS_CUDA_TRY(cudaStreamWaitEvent(as, un.ev_gathered, 0));
    } else {
      if (ts && (rc = trec(ts->gathered, cs))) return rc;
      POS_CUDA_TRY(cudaEventRecord(un.ev_gathered, cs));
      POS_CUDA_TRY(cudaStreamWaitEvent(as, un.ev_gathered, 0));
    }
    // Move(CPU2GPU) analogue: A4 + A4b on the apply stream, once b^l no longer reads W
    if (un.kind == POS_KIND_FC && ev_wfree != l0.ev_in)
      POS_CUDA_TRY(cudaStreamWaitEvent(as, ev_wfree, 0));
    if (ts && (rc = trec(ts->a0, as))) return rc;
    if ((rc = ensure_plan(s, un))) return rc;
    if (un.has_plan) {
      SfbTcPlan pl = un.plan;
      pl.trace = unit_trace(s, un);
      pl.group = group_trace(s, POS_SCHEME_SFB);
      cudaError_t e2 = sfb_tc_launch(pl, s->alpha, 1, as);   // bias fused
      if (e2 != cudaSuccess) return ctx_cuda_fail(c, e2, "reconstruct launch");
    } else {
      rc = reconstruct_apply(un.M, un.N, un.K * P, un.dtype, un.gbuf, 1, un.W, un.N, un.b,
                             s->alpha, c->max_ctas, as);
      if (rc != POS_OK) { if (c->sticky == POS_OK) c->sticky = rc; return rc; }
    }
    if (ts && (rc = trec(ts->a1, as))) return rc;
    if (ts && (rc = trec(ts->done, as))) return rc;
    POS_CUDA_TRY(cudaEventRecord(un.ev_done, as));
  } else {
    if (un.kind == POS_KIND_FC) {
      // FC layer on the PS path: local dense gradient from the factors first
      rc = stage_fc_local_grad(c, un.M, un.N, un.K, un.in_dtype, un.dtype, un.u, un.v, un.gbuf,
                               un.grad, un.b != nullptr, cs);
      if (rc != POS_OK) return rc;
      if (ev_wfree != l0.ev_in) POS_CUDA_TRY(cudaStreamWaitEvent(cs, ev_wfree, 0));
    }
    if (ts && (rc = trec(ts->packed, cs))) return rc;
    bool deferred = false;
    rc = stage_ps_dense(c, un.n, un.grad, un.W, s->alpha, cs, ts ? ts->a0 : nullptr,
                        ts ? ts->a1 : nullptr, /*zero_tail=*/false, unit_trace(s, un),
                        group_trace(s, POS_SCHEME_PS), lane, un.ce_buf, un.exit_word, &deferred);
    if (rc != POS_OK) return rc;
    if (deferred) {
      // the lane's next unit starts right away; the unit is complete once every rank's shard has
      // landed, which the exit wait on the completion stream establishes
      cudaStream_t ds = s->pool[7];
      POS_CUDA_TRY(cudaEventRecord(un.ev_issued, cs));
      POS_CUDA_TRY(cudaStreamWaitEvent(ds, un.ev_issued, 0));
      if ((rc = symm_ps_exit_wait(c, un.exit_word, lane, ds))) return rc;
      if (ts && (rc = trec(ts->done, ds))) return rc;
      POS_CUDA_TRY(cudaEventRecord(un.ev_done, ds));
    } else {
      if (ts && (rc = trec(ts->done, cs))) return rc;
      POS_CUDA_TRY(cudaEventRecord(un.ev_done, cs));
    }
  }
  return POS_OK;
}

int check_layer(pos_sched* s, int32_t l) {
  POS_CHECK_ARG(s, "NULL scheduler");
  POS_CHECK_ARG(l >= 0 && l < s->L, "layer %d out of [0, %d)", l, s->L);
  return POS_OK;
}

int trigger(pos_sched* s, int32_t l, cudaEvent_t ev_in, cudaEvent_t ev_wfree) {
  Layer& ly = s->layers[l];
  if (!s->in_iter) POS_FAIL(POS_ESTATE, "trigger of layer %d outside begin/end", l);
  if (ly.triggered) POS_FAIL(POS_ESTATE, "layer %d triggered twice in one iteration", l);
  ly.ev_in = ev_in;
  ly.ev_wfree = ev_wfree;
  ly.triggered = true;
  s->n_triggered++;
  Unit& un = s->units[ly.unit];
  if (--un.pending > 0) return POS_OK;      // bucket: wait for its remaining layers
  s->order.push_back(ly.unit);
  if (s->flags & POS_SCHED_SEQUENTIAL) return POS_OK;  // deferred to pos_sched_end
  return issue_unit(s, ly.unit);
}

int new_unit(pos_sched* s, Unit&& u, int* out) {
  const bool tf = timing_full(s), ta = timing_any(s);
  int rc;
  if ((rc = make_event(&u.ev_gathered, false)) || (rc = make_event(&u.ev_done, false))) return rc;
  pos_ctx* c = s->ctx;
  if (u.scheme == POS_SCHEME_PS && s->defer_exit && c->world > 1 && !c->local) {
    POS_CUDA_TRY(cudaMalloc(&u.exit_word, sizeof(uint32_t)));
    POS_CUDA_TRY(cudaMemset(u.exit_word, 0, sizeof(uint32_t)));
    if ((rc = make_event(&u.ev_issued, false))) return rc;
  }
  if (u.scheme == POS_SCHEME_PS && c->ps_ce && c->world > 1 && !c->local &&
      (s->flags & POS_SCHED_NO_SYMM) == 0 &&
      symm_lookup(c, u.W, (size_t)pos_padded_size(u.n, c->world) * 4)) {
    // collective (every rank registers the same units in the same order, and the test above
    // depends on rank-invariant registration only)
    if ((rc = pos_mem_alloc(c, symm_ce_bytes(u.n, c->world), &u.ce_buf))) return rc;
  }
  if (ta)
    for (auto& t : u.ring) {
      if ((rc = make_event(&t.a0, true)) || (rc = make_event(&t.a1, true))) return rc;
      if (tf && ((rc = make_event(&t.start, true)) || (rc = make_event(&t.packed, true)) ||
                 (rc = make_event(&t.gathered, true)) || (rc = make_event(&t.done, true))))
        return rc;
    }
  u.seq = (int)s->units.size();
  s->units.push_back(std::move(u));
  *out = (int)s->units.size() - 1;
  return POS_OK;
}

int add_layer(pos_sched* s, int32_t l, int kind, int unit) {
  Layer& ly = s->layers[l];
  ly.kind = kind;
  ly.unit = unit;
  ly.added = true;
  return POS_OK;
}

int check_add(pos_sched* s, int32_t l) {
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (s->in_iter) POS_FAIL(POS_ESTATE, "add after begin");
  if (s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d added twice", l);
  return POS_OK;
}

}  // namespace

extern "C" {

int pos_sched_create(pos_ctx* c, int32_t n_layers, int32_t flags, pos_sched** out) {
  clear_error();
  POS_CHECK_ARG(c && out, "NULL argument");
  POS_CHECK_ARG(n_layers >= 1, "n_layers must be >= 1");
  POS_CHECK_ARG((flags & ~(POS_SCHED_TIMING | POS_SCHED_SEQUENTIAL | POS_SCHED_TIMING_APPLY |
                            POS_SCHED_NO_SYMM | POS_SCHED_PS_AFTER_SFB |
                            POS_SCHED_STATIC_TILES | POS_SCHED_TRACE)) == 0,
                "unknown flags");
  POS_CHECK_ARG(!c->local || c->world == 1, "the scheduler needs a real (or 1-worker) context");
  pos_sched* s = new pos_sched();
  s->ctx = c;
  s->L = n_layers;
  s->flags = flags;
  s->ps_after_sfb = (flags & POS_SCHED_PS_AFTER_SFB) != 0;
  if (const char* e = getenv("POS_SFB_STREAMS")) s->sfb_streams = std::max(1, std::min(3, atoi(e)));
  if (const char* e = getenv("POS_PACK_STREAM")) s->pack_stream = e[0] == '1' ? 1 : 0;
  if (const char* e = getenv("POS_PS_DEFER")) s->defer_exit = e[0] != '0';
  s->layers.resize(n_layers);
  s->units.reserve(n_layers);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  for (int i = 0; i < kPool; ++i) {
    cudaError_t e = cudaStreamCreateWithPriority(&s->pool[i], cudaStreamNonBlocking,
                                                 (i == 5 || i == 7) ? hi : lo);
    if (e != cudaSuccess) { pos_sched_destroy(s); return ctx_cuda_fail(c, e, "stream create"); }
  }
  if (cudaEventCreateWithFlags(&s->ev_end, cudaEventDisableTiming) != cudaSuccess) {
    pos_sched_destroy(s);
    POS_FAIL(POS_ECUDA, "event create failed");
  }
  *out = s;
  return POS_OK;
}

int pos_sched_add_fc(pos_sched* s, int32_t l, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                     int32_t dtype, float* W, float* b, float* grad, int32_t force_scheme) {
  clear_error();
  int rc = check_add(s, l);
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
  // Every rank must reconstruct with the same kernel (tensor-core vs SIMT results differ in the
  // last bits) and pick the same gather protocol: decide from rank-invariant inputs only, and
  // reject a W the tensor-core plan cannot address instead of silently falling back on one rank.
  if (c->world > 1 && scheme == POS_SCHEME_SFB && (N % 4) == 0)
    POS_CHECK_ARG(aligned16(W), "W must be 16-byte aligned (P > 1, tensor-core reconstruction)");
  if (scheme == POS_SCHEME_PS) {
    POS_CHECK_ARG(grad, "FC layer on the PS path needs a grad buffer");
    POS_CHECK_ARG(!b || b == W + M * N, "FC layer on the PS path needs b == W + M*N");
    POS_CHECK_ARG(aligned16(W) && aligned16(grad), "W and grad must be 16-byte aligned");
  }
  Unit u;
  u.kind = POS_KIND_FC;
  u.scheme = scheme;
  u.M = M; u.N = N; u.K = K; u.n = n;
  u.in_dtype = in_dtype; u.dtype = dtype;
  u.W = W; u.b = b; u.grad = grad;
  u.members = {l};
  if (scheme == POS_SCHEME_SFB) {
    u.sfb_idx = s->n_sfb++;
    if (sfb_tc_would_pair(K * c->world * rows_per_sample(dtype), c->world == 1)) s->any_pair = true;
  }
  const int64_t rows = (scheme == POS_SCHEME_SFB ? K * c->world : K) * rows_per_sample(dtype);
  size_t bytes = (size_t)(rows * row_elems(M, N) * dtype_bytes(dtype));
  if (scheme == POS_SCHEME_SFB && c->world > 1 && !c->local && (s->flags & POS_SCHED_NO_SYMM) == 0) {
    // gather buffer in symmetric memory: the factors are multicast straight into it (collective,
    // every rank registers its layers in the same order). Flag mode (tensor-core path only: the
    // reconstruction selects the buffer on the device): two buffers + P ready flags in one
    // allocation.
    const bool fm = gather_flag_mode(dtype, N);
    const size_t al = (bytes + 255) & ~size_t(255);
    const size_t total = fm ? 2 * al + 256 : bytes;
    if (pos_mem_alloc(c, (int64_t)total, &u.gbuf) == POS_OK) {
      u.gbuf_symm = true;
      if (fm) {
        u.flag_mode = true;
        u.gbuf2 = static_cast<uint8_t*>(u.gbuf) + al;
        u.gflags = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(u.gbuf) + 2 * al);
        POS_CUDA_TRY(cudaMalloc(&u.gstate, 2 * sizeof(unsigned)));
        POS_CUDA_TRY(cudaMemset(u.gstate, 0, 2 * sizeof(unsigned)));
      }
    } else {
      clear_error();
    }
  }
  if (!u.gbuf) {
    cudaError_t e = cudaMalloc(&u.gbuf, bytes);
    if (e != cudaSuccess) { (void)cudaGetLastError(); POS_FAIL(POS_ENOMEM, "cudaMalloc(%zu)", bytes); }
  }
  if (scheme == POS_SCHEME_SFB) {   // all launches of this unit run on one stream, in order
    POS_CUDA_TRY(cudaMalloc(&u.tile_counter, 2 * sizeof(unsigned int)));
    POS_CUDA_TRY(cudaMemset(u.tile_counter, 0, 2 * sizeof(unsigned int)));
  }
  if (scheme == POS_SCHEME_PS) {
    const int64_t padded = pos_padded_size(n, c->world);
    if (padded > n) POS_CUDA_TRY(cudaMemset(grad + n, 0, (size_t)(padded - n) * sizeof(float)));
  }
  int ui;
  if ((rc = new_unit(s, std::move(u), &ui)) || (rc = add_layer(s, l, POS_KIND_FC, ui))) return rc;
  return scheme;
}

int pos_sched_add_dense_bucket(pos_sched* s, int32_t l_first, int32_t count, const int64_t* n,
                               float* W, float* grad) {
  clear_error();
  POS_CHECK_ARG(s && n && count >= 1, "bad arguments");
  POS_CHECK_ARG(W && grad && aligned16(W) && aligned16(grad), "W, grad: non-NULL, 16-byte aligned");
  int64_t total = 0;
  for (int i = 0; i < count; ++i) {
    int rc = check_add(s, l_first + i);
    if (rc) return rc;
    POS_CHECK_ARG(n[i] >= 1, "layer %d: n must be >= 1", l_first + i);
    total += n[i];
  }
  Unit u;
  u.kind = POS_KIND_DENSE;
  u.scheme = POS_SCHEME_PS;
  u.n = total;
  u.W = W; u.grad = grad;
  for (int i = 0; i < count; ++i) u.members.push_back(l_first + i);
  const int64_t padded = pos_padded_size(total, s->ctx->world);
  if (padded > total)
    POS_CUDA_TRY(cudaMemset(grad + total, 0, (size_t)(padded - total) * sizeof(float)));
  int ui, rc;
  if ((rc = new_unit(s, std::move(u), &ui))) return rc;
  for (int i = 0; i < count; ++i)
    if ((rc = add_layer(s, l_first + i, POS_KIND_DENSE, ui))) return rc;
  return POS_SCHEME_PS;
}

int pos_sched_add_dense(pos_sched* s, int32_t l, int64_t n, float* W, float* grad) {
  return pos_sched_add_dense_bucket(s, l, 1, &n, W, grad);
}

int pos_sched_begin(pos_sched* s, float alpha) {
  clear_error();
  POS_CHECK_ARG(s, "NULL scheduler");
  if (s->in_iter) POS_FAIL(POS_ESTATE, "begin twice without end");
  for (int l = 0; l < s->L; ++l)
    if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d was never added", l);
  int rc = ctx_check(s->ctx);
  if (rc) return rc;
  if (tracing(s) && (rc = prepare_tracing(s))) return rc;
  if (s->pack_stream < 0) {
    // Which chain is the long pole: the PS units' NVLink transfers or the reconstructions' HBM
    // streams? If the PS chain is, the factor packs leave the comm stream so the first PS unit
    // starts at once (measured, P = 2 / 4: VGG19 -9% / -5%, Inception-V3 -5% / -4%); otherwise
    // they stay ahead of the PS units so every reconstruction can start early (VGG19-22K +2% / +5%,
    // AlexNet +14% / +25% with the packs moved). Rank-invariant: registered units only.
    // per-direction NVLink rate of the fused PS units / NCCL (profiles/nvlink_peaks.json: 452 GB/s
    // at P = 2, 671 at P = 4; P = 8 unmeasured, taken as P = 4's) and the measured HBM copy rate
    const double P = (double)s->ctx->world;
    const double kNvlBps = s->ctx->world == 2 ? 452e9 : 671e9, kHbmBps = 6551e9;
    double t_ps = 0.0, t_sfb = 0.0;
    for (const auto& un : s->units) {
      if (un.scheme == POS_SCHEME_SFB) t_sfb += 8.0 * (double)un.M * (double)un.N / kHbmBps;
      else t_ps += 8.0 * (P - 1.0) / P * (double)un.n / kNvlBps;
    }
    s->pack_stream = t_ps > t_sfb ? 1 : 0;
  }
  if (s->lanes == 0) {
    // Two PS lanes pay off only when the PS units dominate the step: P = 4 Inception-V3 -6% (SFB
    // parameters 0.12x the PS ones), but VGG19 +22% (6x), VGG19-22K +10% (10x) — the second lane's
    // units then slow the reconstructions
    int n_ps = 0;
    double t_ps = 0.0, t_sfb = 0.0;
    for (const auto& un : s->units) {
      if (un.scheme == POS_SCHEME_SFB) t_sfb += 8.0 * (double)un.M * (double)un.N;
      else { t_ps += 8.0 * (double)un.n; ++n_ps; }
    }
    s->lanes = s->ctx->ps_lanes > 0 ? s->ctx->ps_lanes
                                    : ((n_ps >= 4 && t_sfb < 0.5 * t_ps) ? 2 : 1);
  }
  for (auto& ly : s->layers) ly.triggered = false;   // C := 0
  for (auto& un : s->units) un.pending = (int)un.members.size();
  s->order.clear();
  s->n_triggered = 0;
  s->last_sfb = -1;
  s->alpha = alpha;
  s->in_iter = true;
  s->iter += 1;
  return POS_OK;
}

int pos_sched_factors_ready(pos_sched* s, int32_t l, int64_t rows, const void* u, const void* v,
                            void* factors_ready, void* weights_free) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  Layer& ly = s->layers[l];
  if (!ly.added || ly.kind != POS_KIND_FC) POS_FAIL(POS_ESTATE, "layer %d is not an FC layer", l);
  POS_CHECK_ARG(u && v, "NULL factors");
  POS_CHECK_ARG(factors_ready, "NULL factors_ready event");
  Unit& un = s->units[ly.unit];
  POS_CHECK_ARG(rows == un.K,
                "layer %d: %lld factor rows but K = %lld was registered (pad a short batch with "
                "zero rows)", l, (long long)rows, (long long)un.K);
  un.u = u;
  un.v = v;
  return trigger(s, l, (cudaEvent_t)factors_ready, (cudaEvent_t)weights_free);
}

int pos_sched_grad_ready(pos_sched* s, int32_t l, void* grad_ready) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  Layer& ly = s->layers[l];
  if (!ly.added || ly.kind != POS_KIND_DENSE) POS_FAIL(POS_ESTATE, "layer %d is not a dense layer", l);
  POS_CHECK_ARG(grad_ready, "NULL grad_ready event");
  return trigger(s, l, (cudaEvent_t)grad_ready, nullptr);
}

int pos_sched_wait_layer(pos_sched* s, int32_t l, void* consumer) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  Layer& ly = s->layers[l];
  if (!ly.added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  if (s->in_iter && s->units[ly.unit].pending > 0)
    POS_FAIL(POS_ESTATE, "the unit of layer %d has not been issued yet", l);
  POS_CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)consumer, s->units[ly.unit].ev_done, 0));
  return POS_OK;
}

static int end_impl(pos_sched* s, cudaStream_t cs, bool wait_all) {
  POS_CHECK_ARG(s, "NULL scheduler");
  if (!s->in_iter) POS_FAIL(POS_ESTATE, "end without begin");
  if (s->n_triggered != s->L) {
    POS_FAIL(POS_ESTATE, "end with %d of %d layers triggered", s->n_triggered, s->L);
  }
  if (s->flags & POS_SCHED_SEQUENTIAL) {
    POS_CUDA_TRY(cudaEventRecord(s->ev_end, cs));
    for (int u : s->order) {
      int rc = issue_unit(s, u);
      if (rc) { s->in_iter = false; return rc; }
    }
  }
  if (wait_all)
    for (auto& un : s->units) POS_CUDA_TRY(cudaStreamWaitEvent(cs, un.ev_done, 0));
  s->in_iter = false;
  return ctx_check(s->ctx);
}

int pos_sched_end(pos_sched* s, void* consumer) {
  clear_error();
  return end_impl(s, (cudaStream_t)consumer, true);
}

int pos_sched_end_layers(pos_sched* s, void* producer) {
  clear_error();
  return end_impl(s, (cudaStream_t)producer, false);
}

int pos_sched_wait(pos_sched* s, int64_t timeout_ms) {
  clear_error();
  POS_CHECK_ARG(s && timeout_ms >= 0, "bad arguments");
  if (s->in_iter) POS_FAIL(POS_ESTATE, "wait inside an iteration (call pos_sched_end first)");
  if (s->captured) POS_FAIL(POS_ESTATE, "iterations were captured into CUDA graphs: synchronise the graph's stream");
  const auto t0 = std::chrono::steady_clock::now();
  for (auto& un : s->units) {
    for (;;) {
      const cudaError_t q = cudaEventQuery(un.ev_done);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) return ctx_cuda_fail(s->ctx, q, "pos_sched_wait");
      int rc = ctx_check(s->ctx);          // a device-side watchdog expiry ends the wait at once
      if (rc) return rc;
      const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(
                          std::chrono::steady_clock::now() - t0).count();
      if (timeout_ms > 0 && ms > timeout_ms)
        POS_FAIL(POS_ETIMEOUT, "pos_sched_wait: iteration not complete after %lld ms",
                 (long long)timeout_ms);
      std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  return ctx_check(s->ctx);
}

int pos_sched_scheme(pos_sched* s, int32_t l) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  return s->units[s->layers[l].unit].scheme;
}

int pos_sched_timing(pos_sched* s, int32_t l, float* pack_ms, float* comm_ms, float* apply_ms) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!timing_any(s)) POS_FAIL(POS_ESTATE, "scheduler created without timing");
  if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  Unit& un = s->units[s->layers[l].unit];
  for (auto& t : un.ring)
    if ((rc = harvest(un, t, s->captured))) return rc;
  if (un.n_acc == 0) POS_FAIL(POS_ESTATE, "no timed iteration of layer %d yet", l);
  if (pack_ms) *pack_ms = (float)(un.acc_pack / un.n_acc);
  if (comm_ms) *comm_ms = (float)(un.acc_comm / un.n_acc);
  if (apply_ms) *apply_ms = (float)(un.acc_apply / un.n_acc);
  return (int)(un.n_acc > INT32_MAX ? INT32_MAX : un.n_acc);
}

int pos_sched_timing_span(pos_sched* s, int32_t scheme, float* span_ms) {
  clear_error();
  POS_CHECK_ARG(s && span_ms, "bad arguments");
  POS_CHECK_ARG(scheme == POS_SCHEME_SFB || scheme == POS_SCHEME_PS, "bad scheme %d", scheme);
  if (!timing_any(s)) POS_FAIL(POS_ESTATE, "scheduler created without timing");
  double acc = 0;
  int n = 0;
  for (int t = 0; t < kTRing; ++t) {
    const TSlot* ref = nullptr;
    bool all = true, any = false;
    for (auto& un : s->units) {
      if (un.scheme != scheme) continue;
      any = true;
      if (!un.ring[t].used) { all = false; break; }
      if (!ref) ref = &un.ring[t];
    }
    if (!any || !all) continue;
    float lo = 0, hi = 0;
    bool first = true;
    for (auto& un : s->units) {
      if (un.scheme != scheme) continue;
      const TSlot& ts = un.ring[t];
      POS_CUDA_TRY(cudaEventSynchronize(ts.a1));
      float a0 = 0, a1 = 0;
      POS_CUDA_TRY(cudaEventElapsedTime(&a0, ref->a0, ts.a0));
      POS_CUDA_TRY(cudaEventElapsedTime(&a1, ref->a0, ts.a1));
      if (first || a0 < lo) lo = a0;
      if (first || a1 > hi) hi = a1;
      first = false;
    }
    acc += hi - lo;
    ++n;
  }
  if (n == 0) POS_FAIL(POS_ESTATE, "no iteration with live timing events for scheme %d", scheme);
  *span_ms = (float)(acc / n);
  return n;
}

int pos_sched_timeline(pos_sched* s, float* out, int32_t max_units) {
  clear_error();
  POS_CHECK_ARG(s && out && max_units >= 0, "bad arguments");
  if (!timing_full(s)) POS_FAIL(POS_ESTATE, "scheduler created without POS_SCHED_TIMING");
  const int nu = (int)s->units.size();
  // the most recent iteration slot that every unit has recorded
  int slot = -1;
  for (int k = 0; k < kTRing && slot < 0; ++k) {
    const int t = (int)(((s->iter - 1 - k) % kTRing + kTRing) % kTRing);
    bool all = true;
    for (auto& un : s->units) all = all && un.ring[t].used;
    if (all) slot = t;
  }
  if (slot < 0) POS_FAIL(POS_ESTATE, "no iteration with live timing events");
  const cudaEvent_t ref = s->units[s->order.empty() ? 0 : s->order[0]].ring[slot].start;
  POS_CUDA_TRY(cudaEventSynchronize(ref));
  for (int u = 0; u < nu && u < max_units; ++u) {
    const TSlot& t = s->units[u].ring[slot];
    const cudaEvent_t ev[6] = {t.start, t.packed, t.gathered, t.a0, t.a1, t.done};
    for (int k = 0; k < 6; ++k) {
      float ms = -1.0f;
      if (ev[k] && !(k == 2 && s->units[u].scheme != POS_SCHEME_SFB)) {
        POS_CUDA_TRY(cudaEventSynchronize(ev[k]));
        POS_CUDA_TRY(cudaEventElapsedTime(&ms, ref, ev[k]));
      }
      out[6 * u + k] = ms;
    }
  }
  return nu;
}

static int read_trace(const unsigned long long* rec, double* avg_us, double* last_us,
                      int64_t* n) {
  unsigned long long h[kTraceWords];
  POS_CUDA_TRY(cudaMemcpy(h, rec, sizeof(h), cudaMemcpyDeviceToHost));
  if (n) *n = (int64_t)h[3];
  if (avg_us) *avg_us = h[3] ? (double)h[4] / (double)h[3] * 1e-3 : 0.0;
  if (last_us) *last_us = h[3] ? (double)(h[6] - h[5]) * 1e-3 : 0.0;
  return POS_OK;
}

int pos_sched_trace(pos_sched* s, int32_t l, double* avg_us, double* last_us, int64_t* launches) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!tracing(s) && s->traced_ctas == -2) POS_FAIL(POS_ESTATE, "tracing was never on (POS_SCHED_TRACE / pos_sched_set_trace)");
  if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  const Unit& un = s->units[s->layers[l].unit];
  if (!un.trace) POS_FAIL(POS_ESTATE, "no traced iteration yet");
  POS_CUDA_TRY(cudaDeviceSynchronize());
  return read_trace(un.trace, avg_us, last_us, launches);
}

int pos_sched_trace_last(pos_sched* s, int32_t l, int64_t* start_ns, int64_t* end_ns) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  POS_CHECK_ARG(start_ns && end_ns, "NULL output");
  if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  const Unit& un = s->units[s->layers[l].unit];
  if (!un.trace) POS_FAIL(POS_ESTATE, "no traced iteration yet");
  POS_CUDA_TRY(cudaDeviceSynchronize());
  unsigned long long h[kTraceWords];
  POS_CUDA_TRY(cudaMemcpy(h, un.trace, sizeof(h), cudaMemcpyDeviceToHost));
  if (h[3] == 0) POS_FAIL(POS_ESTATE, "no traced launch of layer %d yet", l);
  *start_ns = (int64_t)h[5];
  *end_ns = (int64_t)h[6];
  return POS_OK;
}

int pos_sched_trace_span(pos_sched* s, int32_t scheme, double* avg_us, int64_t* steps) {
  clear_error();
  POS_CHECK_ARG(s && (scheme == POS_SCHEME_SFB || scheme == POS_SCHEME_PS), "bad arguments");
  if (!tracing(s) && s->traced_ctas == -2) POS_FAIL(POS_ESTATE, "tracing was never on (POS_SCHED_TRACE / pos_sched_set_trace)");
  const int k = scheme == POS_SCHEME_SFB ? 1 : 0;
  if (!s->group[k] || s->group_expected[k] == 0)
    POS_FAIL(POS_ESTATE, "no traced group for scheme %d (no units, or an untraced SIMT path)", scheme);
  POS_CUDA_TRY(cudaDeviceSynchronize());
  return read_trace(s->group[k], avg_us, nullptr, steps);
}

int pos_sched_trace_reset(pos_sched* s) {
  clear_error();
  POS_CHECK_ARG(s, "bad arguments");
  if (!tracing(s) && s->traced_ctas == -2) POS_FAIL(POS_ESTATE, "tracing was never on (POS_SCHED_TRACE / pos_sched_set_trace)");
  POS_CUDA_TRY(cudaDeviceSynchronize());
  for (auto& un : s->units)
    if (un.trace) POS_CUDA_TRY(ktrace_reset(un.trace));
  for (auto* g : s->group)
    if (g) POS_CUDA_TRY(ktrace_reset(g));
  return POS_OK;
}

int pos_sched_set_trace(pos_sched* s, int32_t on) {
  clear_error();
  POS_CHECK_ARG(s, "bad arguments");
  if (s->in_iter) POS_FAIL(POS_ESTATE, "pos_sched_set_trace inside an iteration");
  if (on) {
    s->flags |= POS_SCHED_TRACE;
    // allocate / re-arm the records now: iteration begin may run under CUDA-graph stream capture
    int rc = prepare_tracing(s);
    if (rc) return rc;
  } else {
    s->flags &= ~POS_SCHED_TRACE;
  }
  return POS_OK;
}

int pos_sched_timing_reset(pos_sched* s) {
  clear_error();
  POS_CHECK_ARG(s, "NULL scheduler");
  if (!timing_any(s)) POS_FAIL(POS_ESTATE, "scheduler created without timing");
  for (auto& un : s->units) {
    if (!s->captured) {                   // eager: retire in-flight slots; graph: keep them live
      for (auto& t : un.ring) {
        int rc = harvest(un, t);
        if (rc) return rc;
      }
    }
    un.acc_pack = un.acc_comm = un.acc_apply = 0;
    un.n_acc = 0;
  }
  return POS_OK;
}

int pos_sched_unit_of(pos_sched* s, int32_t l) {
  clear_error();
  int rc = check_layer(s, l);
  if (rc) return rc;
  if (!s->layers[l].added) POS_FAIL(POS_ESTATE, "layer %d not added", l);
  return s->layers[l].unit;
}

int pos_sched_destroy(pos_sched* s) {
  clear_error();
  if (!s) return POS_OK;
  for (auto& un : s->units) {
    if (un.ev_done) cudaEventSynchronize(un.ev_done);
    if (un.ev_gathered) cudaEventDestroy(un.ev_gathered);
    if (un.ev_done) cudaEventDestroy(un.ev_done);
    for (auto& t : un.ring) {
      cudaEvent_t te[] = {t.start, t.packed, t.gathered, t.a0, t.a1, t.done};
      for (cudaEvent_t e : te)
        if (e) cudaEventDestroy(e);
    }
    if (un.gbuf) {
      if (un.gbuf_symm) pos_mem_free(s->ctx, un.gbuf);
      else cudaFree(un.gbuf);
    }
    if (un.tile_counter) cudaFree(un.tile_counter);
    if (un.trace) cudaFree(un.trace);
    if (un.gstate) cudaFree(un.gstate);
    if (un.ce_buf) pos_mem_free(s->ctx, un.ce_buf);
    if (un.exit_word) cudaFree(un.exit_word);
    if (un.ev_issued) cudaEventDestroy(un.ev_issued);
  }
  for (auto st : s->pool)
    if (st) cudaStreamDestroy(st);
  if (s->ev_end) cudaEventDestroy(s->ev_end);
  for (auto* g : s->group)
    if (g) cudaFree(g);
  delete s;
  return POS_OK;
}

}  // extern "C"
