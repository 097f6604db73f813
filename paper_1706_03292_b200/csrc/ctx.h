// Internal definition of the context (pos_ctx) shared by ctx.cpp and sched.cpp.
#pragma once

#include <nccl.h>

#include "common.h"

struct pos_ctx {
  int world = 1;         // number of workers P (real ranks, or simulated for pos_init_local)
  int rank = 0;
  int device = 0;
  bool local = false;    // pos_init_local: simulated P, no NCCL
  ncclComm_t comm = nullptr;
  cudaStream_t comm_stream = nullptr;  // high-priority stream for collectives (scheduler)
  // fused PS units may run on up to kMaxLanes concurrent LANES: each lane has its own stream and
  // its own cross-GPU barrier slots / epoch, so units of different lanes overlap while each lane
  // stays stream-ordered (POS_PS_LANES; the scheduler assigns lanes by unit registration order)
  cudaStream_t lane_stream[2] = {nullptr, nullptr};   // [0] = comm_stream
  int ps_lanes = 0;    // 1 / 2 forced (POS_PS_LANES), 0 = the scheduler decides
  int max_ctas = 0;
  void* ws = nullptr;    // one-shot workspace (grow-only)
  size_t ws_bytes = 0;
  int sticky = POS_OK;   // first asynchronous error seen
  void* symm = nullptr;  // symmetric-memory state (symm.cu): NCCL device comm + windows
  // watchdog: every cross-GPU wait in a kernel gives up after timeout_ns (0 = unbounded) and
  // writes a site code into this host-mapped word (first error wins); read without a sync
  volatile int* err_host = nullptr;
  int* err_dev = nullptr;
  unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
  int reduce_order = POS_REDUCE_AUTO;     // PS reduce: NVLS switch order, fixed rank order, auto
  // PS transport of scheduler units (POS_PS_CE): 1 = the copy engines move the gradient pieces and
  // the fresh shards (symm_ps_ce), 0 = the SM-driven fused kernel (symm_ps_fused). Fixed at context
  // creation: the scheduler allocates the receive buffers at registration.
  int ps_ce = 0;
  int fault = POS_FAULT_NONE, fault_rank = -1;   // fault injection (tests)
};

namespace pos {

// grow-only workspace; synchronises the device when it has to reallocate
int ctx_workspace(pos_ctx* c, size_t bytes, void** out);
// record a CUDA / NCCL failure as sticky and format the message
int ctx_cuda_fail(pos_ctx* c, cudaError_t e, const char* what);
int ctx_nccl_fail(pos_ctx* c, ncclResult_t r, const char* what);
// polls the communicator for asynchronous errors (sticky)
int ctx_check(pos_ctx* c);

inline ncclDataType_t nccl_type(int32_t dtype) {
  return dtype == POS_DT_BF16 ? ncclBfloat16 : ncclFloat32;
}

// stages shared by the one-shot entry points and the scheduler
// zero_tail: zero grad[n, P*S) first (the one-shot API; the scheduler zeroes it once at add time
// and the tail stays zero because the in-place reduce-scatter only ever sums zeros into it).
// ce_buf: the unit's copy-engine receive buffer (symm_ce_bytes, from pos_mem_alloc) or nullptr
// exit_word: defer the fused kernel's exit barrier (symm_ps_fused); *deferred tells whether it was
int stage_ps_dense(pos_ctx* c, int64_t n, float* grad, float* W, float alpha, cudaStream_t s,
                   cudaEvent_t ev_rs_done, cudaEvent_t ev_apply_done, bool zero_tail,
                   KTrace tr = {}, KTrace tg = {}, int lane = 0, void* ce_buf = nullptr,
                   uint32_t* exit_word = nullptr, bool* deferred = nullptr);
// grid of the traced kernel stage_ps_dense launches for a unit of n parameters on this rank
int ps_stage_grid(pos_ctx* c, int64_t n, float* grad, float* W, void* ce_buf = nullptr);
int stage_fc_local_grad(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                        int32_t dtype, const void* u, const void* v, void* pack_buf, float* grad,
                        int32_t has_bias, cudaStream_t s);

// symmetric-memory (NVLS) path, symm.cu
void symm_destroy(pos_ctx* c);
// fused reduce-scatter + apply + all-gather over NVLS when grad and W are symmetric; *done = false
// (and nothing enqueued) otherwise
// exit_word != nullptr: deferred exit (the kernel writes its epoch there; the caller completes the
// unit with symm_ps_exit_wait on another stream, stream-ordered after this launch)
int symm_ps_fused(pos_ctx* c, int64_t n, float* grad, float* W, float alpha, cudaStream_t s,
                  cudaEvent_t ev_a0, cudaEvent_t ev_a1, bool* done, KTrace tr = {},
                  KTrace tg = {}, int lane = 0, uint32_t* exit_word = nullptr);
int symm_ps_exit_wait(pos_ctx* c, const uint32_t* exit_word, int lane, cudaStream_t s);
constexpr int kMaxLanes = 2;
// Copy-engine PS unit (POS_PS_CE): A6 as copy-engine pushes of this rank's gradient pieces into
// their owners' receive buffers, A7 as a local kernel summing the P pieces in rank order into the
// owned shard of W, A8 as copy-engine pushes of the fresh shard into every replica; completion is
// signalled with release flags in the receive buffer's window and awaited with bounded polls.
// Needs W (padded) symmetric and ce_buf = a symmetric allocation of symm_ce_bytes(n, P) bytes (one
// per unit: the flags are reset-style, safe because a unit's iterations are stream-ordered on
// every rank). *done = false (nothing enqueued) otherwise.
int symm_ps_ce(pos_ctx* c, int64_t n, float* grad, float* W, void* ce_buf, float alpha,
               cudaStream_t s, cudaEvent_t ev_a0, cudaEvent_t ev_a1, bool* done, KTrace tr = {},
               KTrace tg = {});
int64_t symm_ce_bytes(int64_t n, int P);
int symm_ce_grid(pos_ctx* c, int64_t n);
// grid of the fused PS kernel for a unit of n parameters (rank-invariant)
int symm_ps_grid(pos_ctx* c, int64_t n);
// pack this rank's factors and multicast them into every rank's gather buffer when the gather
// buffer is symmetric; *done = false otherwise. Barrier mode (gbuf2 == nullptr): entry + exit
// barriers. Flag mode: gbuf / gbuf2 double buffer (by iteration parity) and the P ready flags, all
// in ONE symmetric allocation; fstate = this rank's device state (2 x u32, zeroed); no waiting —
// the consumer calls symm_wait_gathered on its stream before reading the gather buffer.
int symm_pack_mc(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                 const void* u, const void* v, void* gbuf, cudaStream_t s, bool* done,
                 void* gbuf2 = nullptr, uint32_t* flags = nullptr, unsigned* fstate = nullptr);
// consumer-side wait (bounded) for the P ready flags of flag mode, before the reconstruction
int symm_wait_gathered(pos_ctx* c, const uint32_t* flags, const unsigned* fstate, int P,
                       cudaStream_t s);
// true if [p, p+bytes) lies inside one symmetric window of the context
bool symm_lookup(pos_ctx* c, const void* p, size_t bytes);
// description of a watchdog site code (error word)
const char* site_name(int site);

}  // namespace pos
