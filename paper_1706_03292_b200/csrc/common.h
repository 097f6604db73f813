// Internal helpers shared by the libposeidon translation units (never installed, never included
// by anything outside csrc/).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "poseidon.h"

#ifdef __CUDACC__
#include <cuda_bf16.h>
#endif

namespace pos {

// thread-local last-error message (pos_last_error)
void set_error(const char* fmt, ...);
void clear_error();

#define POS_FAIL(code, ...)          \
  do {                               \
    ::pos::set_error(__VA_ARGS__);   \
    return (code);                   \
  } while (0)

#define POS_CHECK_ARG(cond, ...)                       \
  do {                                                 \
    if (!(cond)) POS_FAIL(POS_EINVAL, __VA_ARGS__);    \
  } while (0)

#define POS_CUDA_TRY(expr)                                                             \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      POS_FAIL(POS_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e),      \
               __FILE__, __LINE__);                                                    \
  } while (0)

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// gathered factor row layout: [u (M_pad) | v (N_pad)], pads of 8 elements (16 B for bf16)
// Pads of 64 elements keep every gathered row and the v part 128-byte aligned, so each 128-byte
// TMA box row is exactly one L2 line (a 16-byte pad made rows straddle lines: 1.25x slower at
// K*P = 1024). N_pad >= N + 1: column N of every v row is the 1.0 "ones column" (fused bias).
inline int64_t m_pad(int64_t M) { return round_up(M, 64); }
inline int64_t n_pad(int64_t N) { return round_up(N + 1, 64); }
inline int64_t row_elems(int64_t M, int64_t N) { return m_pad(M) + n_pad(N); }
inline int64_t dtype_bytes(int32_t dtype) { return dtype == POS_DT_BF16 ? 2 : 4; }
// Gathered rows per sufficient-factor pair. POS_DT_F32 runs as 3xTF32 on the tensor cores
// (reading S16): the pack writes each pair three times, as K-row blocks (hi u, hi v),
// (hi u, lo v), (lo u, hi v) with hi = tf32(x), lo = tf32(x - hi), so one tf32 contraction over
// 3K rows per slot gives sum_k hi·hi + hi·lo + lo·hi = u_k^T v_k up to the dropped lo·lo term.
// POS_F32_FFMA=1 (read once per process) keeps the rounds-1/2 exact-fp32 mode instead: one row per
// pair and the SIMT FFMA reconstruction.
inline bool f32_ffma() {
  static const bool v = [] {
    const char* e = getenv("POS_F32_FFMA");
    return e && e[0] == '1';
  }();
  return v;
}
inline int64_t rows_per_sample(int32_t dtype) { return dtype == POS_DT_F32 && !f32_ffma() ? 3 : 1; }

int num_sms();

// Lazy module loading (the CUDA 12 default) loads a kernel at its first launch, and a load may have
// to synchronise the context — fatal for kernels that spin on other GPUs' progress (the PS
// barriers, the gather-flag wait): a rank blocked in a load while its own spinning kernel waits for
// a peer that is blocked the same way only resolves through the watchdog. Every kernel of the
// library is therefore loaded when a context is created (cudaFuncGetAttributes forces the load).
cudaError_t preload_mem_kernels();
cudaError_t preload_sfb_kernels();
cudaError_t preload_symm_kernels();

// Kernel launches report errors only through the runtime's last-error state, which other runtime
// or NCCL calls may have left set (non-sticky, already reported to their callers). Clear it right
// before launching so the check after the launch sees only the launch's own error; sticky device
// faults are unaffected (every later call keeps returning them).
inline void clear_stale_launch_error() { (void)cudaGetLastError(); }

// Record a TIMING event: a plain record outside stream capture; an external event node inside a
// capture, so that it remains a real record when the CUDA graph is replayed.
inline cudaError_t record_timing_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  cudaError_t q = cudaStreamIsCapturing(s, &st);
  if (q != cudaSuccess) return q;
  return st == cudaStreamCaptureStatusActive
             ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
             : cudaEventRecord(e, s);
}

// ---- device-side launch trace (SURVEY §5 tracing) ----
// Kernels stamp %globaltimer into a record in device memory instead of the host bracketing them
// with CUDA events (inside a CUDA graph every event record is one more node on the critical
// stream). An INTERVAL is `expected` CTAs: one launch (its grid) or a group of launches (the sum of
// their grids, e.g. all reconstructions of one step). Record words (u64):
//   [0] earliest CTA start of the interval in progress (~0 = none)   [1] latest CTA end
//   [2] CTAs finished                                               [3] intervals completed
//   [4] sum of interval durations (ns)                              [5], [6] last interval's start, end
struct KTrace {
  unsigned long long* rec = nullptr;   // nullptr = tracing off
  unsigned expected = 0;
};
constexpr int kTraceWords = 8;
// allocate / re-arm a record (host)
cudaError_t ktrace_alloc(unsigned long long** rec);
cudaError_t ktrace_reset(unsigned long long* rec);

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long ktrace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// thread 0 of every CTA, first thing
__device__ __forceinline__ void ktrace_begin(const KTrace& t) {
  if (t.rec && threadIdx.x == 0) atomicMin(t.rec, ktrace_now());
}
// thread 0 of every CTA, after the whole CTA's work (callers __syncthreads() first); the last CTA
// of the interval folds it into the sums and re-arms the record
__device__ __forceinline__ void ktrace_end(const KTrace& t) {
  if (!t.rec || threadIdx.x != 0) return;
  atomicMax(t.rec + 1, ktrace_now());
  __threadfence();
  if (atomicAdd(t.rec + 2, 1ull) == (unsigned long long)t.expected - 1) {
    __threadfence();
    const unsigned long long s = atomicOr(t.rec + 0, 0ull), e = atomicOr(t.rec + 1, 0ull);
    t.rec[5] = s;
    t.rec[6] = e;
    t.rec[4] += e > s ? e - s : 0;
    t.rec[3] += 1;
    atomicExch(t.rec + 0, ~0ull);
    atomicExch(t.rec + 1, 0ull);
    atomicExch(t.rec + 2, 0ull);
    __threadfence();
  }
}

// ---- A2 factor pack: one 16-byte output vector of a gathered row ----
// Output elements idx .. idx+VEC-1 of the u or v part (VEC = 8 bf16 / 4 fp32); src = the input row
// (u_k or v_k), lim = its length (M or N), onec = the ones column (N for the v part, -1 for u).
// Chunks entirely inside the row whose source is suitably aligned take vector loads (16 B for
// 8 bf16 / 4 fp32 inputs, 2 x 16 B for 8 fp32 inputs, 8 B for 4 bf16 inputs); the row tail, the
// pad and unaligned rows (M or N not a multiple of the vector) take element loads.
__device__ __forceinline__ float pack_ld1(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float pack_ld1(const float* p) { return *p; }
template <typename Tin, bool kBF16>
__device__ __forceinline__ uint4 pack_chunk(const Tin* __restrict__ src, int64_t idx, int64_t lim,
                                            int64_t onec) {
  constexpr int VEC = kBF16 ? 8 : 4;
  const Tin* p = src + idx;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  if (idx + VEC <= lim) {
    if constexpr (kBF16 && sizeof(Tin) == 2) {          // bf16 -> bf16: a straight copy
      if ((a & 15u) == 0) return __ldg(reinterpret_cast<const uint4*>(p));
    } else if constexpr (kBF16) {                        // fp32 -> bf16
      if ((a & 15u) == 0) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(p));
        const float4 y = __ldg(reinterpret_cast<const float4*>(p) + 1);
        uint4 o;
        __nv_bfloat162 h;
        h = __floats2bfloat162_rn(x.x, x.y); o.x = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(x.z, x.w); o.y = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(y.x, y.y); o.z = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(y.z, y.w); o.w = *reinterpret_cast<uint32_t*>(&h);
        return o;
      }
    } else if constexpr (sizeof(Tin) == 4) {             // fp32 -> fp32
      if ((a & 15u) == 0) return __ldg(reinterpret_cast<const uint4*>(p));
    } else {                                             // bf16 -> fp32
      if ((a & 7u) == 0) {
        const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
        uint4 o;
        o.x = x.x << 16; o.y = x.x & 0xFFFF0000u;
        o.z = x.y << 16; o.w = x.y & 0xFFFF0000u;
        return o;
      }
    }
  }
  uint4 o;
  if constexpr (kBF16) {
    __align__(16) __nv_bfloat16 h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      h[i] = __float2bfloat16_rn(idx + i < lim ? pack_ld1(p + i) : (idx + i == onec ? 1.f : 0.f));
    o = *reinterpret_cast<const uint4*>(h);
  } else {
    float f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      f[i] = idx + i < lim ? pack_ld1(p + i) : (idx + i == onec ? 1.f : 0.f);
    o = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                   __float_as_uint(f[3]));
  }
  return o;
}

// 3xTF32 split (POS_DT_F32): part 1 = tf32 head (round to nearest, ties away), part 2 = the fp32
// remainder x - head, itself rounded to tf32 (the tensor core reads only tf32 bits). 1.0 (the ones
// column) splits into 1 + 0 and 0 into 0 + 0, so the ones column is 1 in blocks 0 and 2 and 0 in
// block 1: the fused bias column sums hi u + lo u = u.
__device__ __forceinline__ float tf32_part(float x, int part) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  if (part == 1) return __uint_as_float(h);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(x - __uint_as_float(h)));
  return __uint_as_float(l);
}
__device__ __forceinline__ uint4 tf32_split4(uint4 q, int part) {
  return make_uint4(__float_as_uint(tf32_part(__uint_as_float(q.x), part)),
                    __float_as_uint(tf32_part(__uint_as_float(q.y), part)),
                    __float_as_uint(tf32_part(__uint_as_float(q.z), part)),
                    __float_as_uint(tf32_part(__uint_as_float(q.w), part)));
}
// gathered row r of a 3xTF32 slot of K pairs: pair r % K, block r / K; the u part is lo in
// block 2, the v part lo in block 1, hi otherwise
__device__ __forceinline__ int split_part(int64_t block, bool v_part) {
  return (v_part ? block == 1 : block == 2) ? 2 : 1;
}
#endif

// ---- kernel launchers (return cudaError_t of the launch) ----
cudaError_t launch_pack_factors(int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                                const void* u, const void* v, void* slot, cudaStream_t s);
// b += alpha * sum_j U[j][m] * V[j][N] over KP gathered ROWS (V[j][N] = the ones column's value)
cudaError_t launch_bias_colsum(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                               int32_t accumulate, float* b, float alpha, cudaStream_t s);
// tr.rec != nullptr: traced; tr.expected = 0 means "this launch alone" (set to its grid)
cudaError_t launch_ps_apply(const float* g, float* W, int64_t count, float alpha, cudaStream_t s,
                            KTrace tr = {}, KTrace tg = {});
// grid of launch_ps_apply's vector kernel for `count` 16-byte-aligned elements (0 = no vector part)
int ps_apply_grid(int64_t count);
constexpr int kMaxSimP = 16;
constexpr int kMaxPeers = 16;   // ranks addressable by the fused symmetric-memory kernels

// Flag-mode (double-buffered, barrier-free) factor gather: decided from RANK-INVARIANT inputs only
// (every rank must make the same choice: it sets the symmetric allocation size and the protocol).
// Tensor-core dtypes with N % 4 == 0 (the reconstruction selects the buffer on the device);
// POS_GATHER_FLAGS=0 turns it off.
inline bool gather_flag_mode(int32_t dtype, int64_t N) {
  static const bool off = [] {
    const char* e = getenv("POS_GATHER_FLAGS");
    return e && e[0] == '0';
  }();
  return !off && dtype != POS_DT_F32 && (N % 4) == 0;
}
cudaError_t launch_sim_ps_reduce_apply(const float* const* grads, int P, float* W, int64_t n,
                                       float alpha, cudaStream_t s);
// SIMT fp32 FFMA reconstruct-and-apply (shapes the TMA path cannot take: N or ldw % 4 != 0,
// unaligned W). KP here = gathered ROWS (samples * rows_per_sample).
cudaError_t launch_sfb_simt(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                            int32_t accumulate, float* W, int64_t ldw, float alpha,
                            cudaStream_t s);
// tcgen05 / TMEM / TMA reconstruct-and-apply (all dtypes; POS_DT_F32 = tf32 kind over the 3xTF32
// rows). KP = SAMPLES (K * P) here and in the plan / pair queries below. Returns
// cudaErrorNotSupported if the shape/alignment cannot use TMA (caller falls back to SIMT).
// b != nullptr: the bias update is fused (needs the ones column of the packed v rows).
cudaError_t launch_sfb_tc(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                          int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                          int max_ctas, cudaStream_t s);
bool sfb_tc_supported(int64_t N, int64_t ldw, const float* W, const void* G);
// the plan for inner dimension KP would use the CTA-pair (cluster) kernel
bool sfb_tc_would_pair(int64_t KP, bool cluster_ok = true);

// A launch plan for the tensor-core reconstruct-and-apply: TMA descriptors encoded once for fixed
// buffers (the scheduler keeps one per SFB layer, so the hot path does no host-side encoding).
struct SfbTcPlan {
  CUtensorMap tmA, tmB, tmW;
  // double-buffered gather (flag mode): maps of the second buffer, selected in the kernel by the
  // parity of (*gsel - 1) (the gather sequence advanced by this rank's pack); gsel == nullptr:
  // always the first buffer
  CUtensorMap tmA2, tmB2;
  const unsigned* gsel = nullptr;
  int64_t M = 0, N = 0, KP = 0;
  int nb_n = 0, num_tiles = 0, nkb = 0, grid = 0;
  bool tf32 = false;
  bool pair = false;       // CTA-pair kernel (cta_group::2, 256-row tiles) — large K*P
  // device scratch (2 x u32, zero-initialised, owned by the plan's creator) for the dynamic tile
  // scheduler; nullptr = static round-robin tiles. Launches sharing a counter must not overlap.
  unsigned int* counter = nullptr;
  float* bias = nullptr;   // fused A4b target (nullptr = no bias)
  KTrace trace, group;     // device-side launch trace of this launch / of a group of launches
};
// false if the shape/alignment/dtype cannot use the tensor-core kernel
bool sfb_tc_make_plan(SfbTcPlan* plan, int64_t M, int64_t N, int64_t KP, int32_t dtype,
                      const void* G, float* W, int64_t ldw, int max_ctas, float* bias = nullptr,
                      const void* G2 = nullptr, bool cluster_ok = true);
cudaError_t sfb_tc_launch(const SfbTcPlan& plan, float alpha, int accumulate, cudaStream_t s);

// A4 + A4b dispatcher used by the C ABI and the context code
int reconstruct_apply(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                      int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                      int max_ctas, cudaStream_t s);

}  // namespace pos
