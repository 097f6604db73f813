// NVLink-SHARP / symmetric-memory path: the PS and SFB collectives fused into
// the kernels that consume them, over NVSwitch multicast (NVLS) memory registered as NCCL symmetric
// windows. NCCL provides only the plumbing (allocation, window registration and the device-side
// address resolution, done ONCE per window here); the data movement, the arithmetic and the
// cross-GPU synchronisation are these kernels.
//
//  * ps_sync_kernel (A6 + A7 + A8 fused): rank r owns shard [lo, hi) of a dense unit.
//      ghat = reduce over ranks of grad[i]    -- (1) workers push gradients; the server sums them
//      w    = W_local[i] + alpha * ghat       -- (2) the server's "apply (+)"
//      store w into W[i] of every replica     -- (3) consistency: every worker reads it back
//    The reduce is either multimem.ld_reduce through the switch (default; the switch picks the
//    summation order) or, in RANK-ORDER mode, plain peer loads summed in rank order 0..P-1
//    (deterministic run to run). The broadcast is a multimem.st (the switch replicates) or P plain
//    stores.
//  * pack_x_kernel (A2 + A3 fused): this rank's sufficient factors, packed and cast, are
//    stored into its slot of EVERY rank's gather buffer (one multicast store, or P unicast stores).
//    Flag mode publishes completion with a release-store of the iteration number into flag[rank]
//    of every replica; the consumer runs wait_flags_kernel before the reconstruction.
//
// Every kernel addresses the other ranks through a POINTER TABLE (per-rank addresses and the
// multicast address, resolved once when a window is registered). The single-GPU LOOPBACK entry
// points at the end of this file run the very same kernels with a table of P local replicas, rank
// after rank in stream order — the driver's one-GPU tests exercise the P > 1 kernel bodies that way.
//
// Cross-GPU waits (entry / exit barriers, gather flags) are bounded: a wait that exceeds the
// context's timeout writes a code into the context's host-mapped error word and the kernel returns;
// the host reports it as the sticky error POS_ETIMEOUT (SURVEY §5 failure detection).
//
// Barriers: per lane, P ENTRY and P EXIT epoch slots (u32) in a symmetric window; slot r holds the
// epoch of rank r's latest kernel instance on the lane. Entry: CTA 0 of each rank multicasts its
// epoch into slot r of every rank; every CTA polls its local slots until all P reach the instance's
// epoch. Exit: each CTA counts itself done; the LAST CTA of the rank multicasts the epoch into the
// exit slots (release) and waits for all P — or, for the scheduler's PS units, records the epoch
// and leaves the wait to xg_exit_wait_kernel on a completion stream, so the next unit of the lane
// starts without a cross-GPU round trip. No CTA waits for a specific CTA of another GPU, so the
// kernels tolerate any residency pattern (a per-CTA-index barrier needs matching CTAs of all GPUs
// co-resident at once). Fused kernels of one lane must be stream-ordered among themselves.
#include <cuda_bf16.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdlib>
#include <vector>

#include "ctx.h"

namespace pos {

struct SymmWindow {
  char* base = nullptr;
  size_t bytes = 0;
  ncclWindow_t win = nullptr;
  char* peer[kMaxPeers] = {};   // every rank's copy of the window (world-rank order)
  char* mc = nullptr;           // multicast (NVLS) address of the window
};

struct SymmState {
  ncclDevComm dev;
  bool ready = false;
  std::vector<SymmWindow> windows;
  SymmWindow bar;                 // internal: [0] entry inbox, [1] exit inbox
  uint32_t* bar_state = nullptr;  // device: [0] entry epoch, [1] exit epoch, [2] CTAs done
};

static SymmState* state(pos_ctx* c) { return static_cast<SymmState*>(c->symm); }

namespace {

// error sites reported through the context's error word (see site_name)
enum { kSitePsEntry = 1, kSitePsExit = 2, kSitePackEntry = 3, kSitePackExit = 4, kSiteFlags = 5,
       kSiteCeData = 6, kSiteCeShard = 7 };

// ------------------------------------------------------------------------------ device -------
__device__ __forceinline__ float4 mm_ld_reduce_v4(const float* p) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ float mm_ld_reduce(const float* p) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void mm_st_v4(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st(float* p, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Spin until *p has reached `target` (mod 2^32). Bounded: after timeout_ns (0 = unbounded) the
// site code is written to the error word (first error wins) and false is returned.
__device__ bool poll_reached(const uint32_t* p, uint32_t target, unsigned long long timeout_ns,
                             int* err, int site) {
  unsigned long long t0 = 0;
  for (uint32_t spin = 1;; ++spin) {
    if ((int32_t)(ld_acquire_sys(p) - target) >= 0) return true;
    if (timeout_ns && (spin & 63) == 0) {
      const unsigned long long t = gtimer();
      if (t0 == 0) {
        t0 = t;
      } else if (t - t0 > timeout_ns) {
        atomicCAS(err, 0, site);
        __threadfence_system();
        return false;
      }
    }
  }
}

// Cross-GPU synchronisation of one fused-kernel instance. local == nullptr: none (P = 1 or the
// single-GPU loopback, where ranks run one after the other in stream order).
// Every lane has a block of slots in the barrier window: entry slots [0, P) and exit slots
// [kXgExit, kXgExit + P); slot r is written only by rank r, with the EPOCH of its latest kernel
// instance on the lane (state[0] + 1: every rank runs the same instances in the same order). A wait
// polls the P slots for >= the instance's epoch, so a rank that has already moved on to a later
// instance still counts as arrived, and no rank can be mistaken for arrived before it was.
struct Xg {
  uint32_t* mc;          // multicast address of this lane's slot block
  uint32_t* local;       // this rank's copy of the slot block
  uint32_t* state;       // [0] epoch of the lane's last instance, [2] CTAs of this instance done
  uint32_t* exit_word;   // deferred exit: the epoch is written here and nobody waits (the caller
                         // runs xg_exit_wait_kernel on another stream); nullptr = wait at exit
  int P, rank;
  unsigned long long timeout_ns;
  int* err;
  int site;              // entry site; exit = site + 1
};
constexpr int kXgExit = kMaxPeers;    // exit slots follow the entry slots
constexpr int kXgLaneBytes = 256;     // slot block of lane k at byte 256 k of the window

// Entry: every rank's inputs (produced by kernels that completed in stream order) are in place.
// The arrival needs no release fence: the data was written by completed kernels.
__device__ __forceinline__ bool xg_enter(const Xg& x) {
  if (!x.local) return true;
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(x.state) + 1u;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    asm volatile("multimem.st.relaxed.sys.global.u32 [%0], %1;" ::"l"(x.mc + x.rank), "r"(e)
                 : "memory");
  int ok = 1;
  if (threadIdx.x < x.P) ok = poll_reached(x.local + threadIdx.x, e, x.timeout_ns, x.err, x.site);
  return __syncthreads_and(ok) != 0;
}

// Exit: the last CTA of this rank (all of the rank's stores performed) publishes the epoch with
// release into every rank's exit slot and — unless the exit is deferred — waits until every rank
// has done the same: every replica's outputs are complete and every input read.
__device__ __forceinline__ void xg_exit(const Xg& x) {
  if (!x.local) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();                 // this CTA's (multicast / peer) stores are performed
    const unsigned prev = atomicAdd(x.state + 2, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      x.state[2] = 0;
      const uint32_t e = x.state[0] + 1u;
      asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(x.mc + kXgExit + x.rank),
                   "r"(e)
                   : "memory");
      if (x.exit_word) {
        *x.exit_word = e;
      } else {
        for (int t = 0; t < x.P; ++t)
          poll_reached(x.local + kXgExit + t, e, x.timeout_ns, x.err, x.site + 1);
      }
      x.state[0] = e;
    }
  }
}

// The deferred exit of one instance (stream-ordered after it): every rank's outputs are complete.
__global__ void xg_exit_wait_kernel(const uint32_t* local, const uint32_t* exit_word, int P,
                                    unsigned long long timeout_ns, int* err, int site) {
  const uint32_t e = *reinterpret_cast<const volatile uint32_t*>(exit_word);
  if (threadIdx.x < P) poll_reached(local + kXgExit + threadIdx.x, e, timeout_ns, err, site);
}

constexpr int kPsThreads = 512;
#ifndef POS_NVLS_UNROLL
#define POS_NVLS_UNROLL 4
#endif
constexpr int kPsUnroll = POS_NVLS_UNROLL;   // 16-byte reductions in flight per thread

// One PS unit on one rank. All pointers address element 0 of the unit's flat buffers.
struct PsArgs {
  const float* g_mc;            // multicast address of grad (kRedMc)
  float* w_mc;                  // multicast address of W (kStMc)
  const float* g[kMaxPeers];    // every rank's grad, rank order (peer reduce)
  float* w[kMaxPeers];          // every rank's W (peer broadcast)
  const float* wl;              // this rank's W
  int P;
  int64_t lo, hi;               // this rank's shard
  float alpha;
  KTrace trace, group;          // device-side launch trace (tracing scheduler)
};

template <bool kRedMc>
__device__ __forceinline__ float4 ps_red4(const PsArgs& a, int64_t i) {
  if constexpr (kRedMc) {
    return mm_ld_reduce_v4(a.g_mc + 4 * i);
  } else {   // fixed rank order: identical on every run, every rank
    float4 s = *reinterpret_cast<const float4*>(a.g[0] + 4 * i);
    for (int p = 1; p < a.P; ++p) {
      const float4 t = *reinterpret_cast<const float4*>(a.g[p] + 4 * i);
      s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
    }
    return s;
  }
}
template <bool kRedMc>
__device__ __forceinline__ float ps_red1(const PsArgs& a, int64_t j) {
  if constexpr (kRedMc) {
    return mm_ld_reduce(a.g_mc + j);
  } else {
    float s = a.g[0][j];
    for (int p = 1; p < a.P; ++p) s += a.g[p][j];
    return s;
  }
}
template <bool kStMc>
__device__ __forceinline__ void ps_st4(const PsArgs& a, int64_t i, float4 v) {
  if constexpr (kStMc) {
    mm_st_v4(a.w_mc + 4 * i, v);
  } else {
    for (int p = 0; p < a.P; ++p) *reinterpret_cast<float4*>(a.w[p] + 4 * i) = v;
  }
}
template <bool kStMc>
__device__ __forceinline__ void ps_st1(const PsArgs& a, int64_t j, float v) {
  if constexpr (kStMc) {
    mm_st(a.w_mc + j, v);
  } else {
    for (int p = 0; p < a.P; ++p) a.w[p][j] = v;
  }
}

template <bool kRedMc, bool kStMc>
// minBlocks 2 caps the registers at 64 per thread, so a PS CTA (512 threads, 32K registers) fits on an
// SM next to a resident reconstruction CTA (256 threads x 120 registers): the fused PS units run
// concurrently with the reconstructions instead of waiting for their SMs to drain
__global__ void __launch_bounds__(kPsThreads, 2) ps_sync_kernel(PsArgs a, Xg x) {
  ktrace_begin(a.trace);
  ktrace_begin(a.group);
  if (!xg_enter(x)) return;
  // lo is a multiple of 64 for a non-empty shard; an empty shard (lo == hi == n, a trailing rank of
  // a small unit) does no work but still takes part in the barriers
  const int64_t v0 = a.lo / 4, v1 = a.lo < a.hi ? a.hi / 4 : v0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = v0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kPsUnroll - 1) * stride < v1; i += kPsUnroll * stride) {
    float4 g[kPsUnroll], w[kPsUnroll];
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      g[u] = ps_red4<kRedMc>(a, i + u * stride);
      w[u] = *reinterpret_cast<const float4*>(a.wl + 4 * (i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      w[u].x = fmaf(a.alpha, g[u].x, w[u].x);
      w[u].y = fmaf(a.alpha, g[u].y, w[u].y);
      w[u].z = fmaf(a.alpha, g[u].z, w[u].z);
      w[u].w = fmaf(a.alpha, g[u].w, w[u].w);
      ps_st4<kStMc>(a, i + u * stride, w[u]);
    }
  }
  for (; i < v1; i += stride) {
    const float4 g = ps_red4<kRedMc>(a, i);
    float4 w = *reinterpret_cast<const float4*>(a.wl + 4 * i);
    w.x = fmaf(a.alpha, g.x, w.x);
    w.y = fmaf(a.alpha, g.y, w.y);
    w.z = fmaf(a.alpha, g.z, w.z);
    w.w = fmaf(a.alpha, g.w, w.w);
    ps_st4<kStMc>(a, i, w);
  }
  if (blockIdx.x == 0)   // scalar tail of the shard
    for (int64_t j = std::max(v1 * 4, a.lo) + threadIdx.x; j < a.hi; j += blockDim.x)
      ps_st1<kStMc>(a, j, fmaf(a.alpha, ps_red1<kRedMc>(a, j), a.wl[j]));
  xg_exit(x);
  if (a.trace.rec || a.group.rec) {
    __syncthreads();
    ktrace_end(a.trace);
    ktrace_end(a.group);
  }
}

// One rank's factor pack + gather. Byte addresses of THIS rank's slot in buffer 0 / 1.
struct PackArgs {
  const void* u;
  const void* v;
  int64_t M, N, Mp, R;
  int64_t K;                     // gathered rows of the slot (pairs * rows_per_sample)
  int64_t Kp;                    // factor pairs
  int split;                     // POS_DT_F32: 3xTF32 blocks (common.h, rows_per_sample)
  char* mc[2];                   // multicast address of the slot (kMc)
  char* dst[2][kMaxPeers];       // the slot in every rank's buffer (unicast / loopback)
  uint32_t* flag_mc;             // multicast address of flag[rank] (flag mode, kMc)
  uint32_t* flag[kMaxPeers];     // flag[rank] in every rank's flags (flag mode, unicast)
  unsigned* state;               // flag mode: this rank's [0] packs completed, [1] CTAs done
  int P;
};

// One 16-byte output vector per thread iteration, into this rank's slot of every rank's buffer.
//  kFlag = false: barrier mode — entry barrier (cross-rank WAR on the single gather buffer: every
//    rank's previous reconstruction has finished reading it) and exit barrier (all P slots landed).
//  kFlag = true: flag mode — no waiting: the gather buffer is double-buffered by the iteration
//    parity read from device memory (a replayed CUDA graph alternates too), and the last CTA to
//    finish publishes "slot of rank r for iteration s is complete" as a release-store of s into
//    flag[r] of every replica. WAR safety: rank r writes buffer s%2 at iteration s only after its
//    iteration s-1 consumed every rank's s-1 flag, and each rank publishes its s-1 flag only after
//    finishing iteration s-2, whose reconstruction was the last reader of buffer s%2.
template <typename Tin, bool kBF16, bool kFlag, bool kMc>
__global__ void __launch_bounds__(256) pack_x_kernel(PackArgs a, Xg x) {
  uint32_t seq = 0;
  if constexpr (!kFlag) {
    if (!xg_enter(x)) return;
  } else {
    seq = *reinterpret_cast<volatile unsigned*>(a.state);
  }
  const int b = (kFlag && (seq & 1)) ? 1 : 0;
  const Tin* u = static_cast<const Tin*>(a.u);
  const Tin* v = static_cast<const Tin*>(a.v);
  constexpr int VEC = kBF16 ? 8 : 4;
  constexpr int EB = kBF16 ? 2 : 4;
  const int64_t chunks_per_row = a.R / VEC, total = a.K * chunks_per_row;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = c / chunks_per_row, col = (c % chunks_per_row) * VEC;
    const int64_t k = a.split ? r % a.Kp : r;     // gathered row r holds factor pair k
    const Tin* src;
    int64_t idx, lim;
    if (col < a.Mp) { src = u + k * a.M; idx = col; lim = a.M; }
    else            { src = v + k * a.N; idx = col - a.Mp; lim = a.N; }
    const int64_t onec = col < a.Mp ? -1 : a.N;   // ones column (fused bias), as in pack_kernel
    uint4 q = pack_chunk<Tin, kBF16>(src, idx, lim, onec);
    if constexpr (!kBF16)
      if (a.split) q = tf32_split4(q, split_part(r / a.Kp, col >= a.Mp));
    const float4 o = make_float4(__uint_as_float(q.x), __uint_as_float(q.y), __uint_as_float(q.z),
                                 __uint_as_float(q.w));   // bit pattern only; stores do not convert
    const int64_t boff = (r * a.R + col) * EB;   // byte offset of this vector in the slot
    if constexpr (kMc) {
      mm_st_v4(reinterpret_cast<float*>(a.mc[b] + boff), o);
    } else {
      for (int p = 0; p < a.P; ++p) *reinterpret_cast<float4*>(a.dst[b][p] + boff) = o;
    }
  }
  if constexpr (!kFlag) {
    xg_exit(x);
  } else {
    __syncthreads();                        // the CTA's stores happen-before thread 0's fence
    if (threadIdx.x == 0) {
      __threadfence_system();
      const unsigned prev = atomicAdd(a.state + 1, 1u);
      if (prev == gridDim.x - 1) {          // last CTA: every CTA's stores are performed
        __threadfence_system();
        a.state[1] = 0;
        a.state[0] = seq + 1;
        if constexpr (kMc) {
          asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(a.flag_mc), "r"(seq + 1)
                       : "memory");
        } else {
          for (int p = 0; p < a.P; ++p)
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flag[p]), "r"(seq + 1)
                         : "memory");
        }
      }
    }
  }
}

// Consumer side of flag mode: returns once every rank's slot of this iteration is in place
// (flag[r] >= this rank's own sequence, which its pack has just advanced). Bounded wait.
__global__ void wait_flags_kernel(const uint32_t* flags, const unsigned* state, int P,
                                  unsigned long long timeout_ns, int* err) {
  const uint32_t want = *reinterpret_cast<const volatile unsigned*>(state);
  for (int r = threadIdx.x; r < P; r += blockDim.x)
    poll_reached(flags + r, want, timeout_ns, err, kSiteFlags);
  __syncthreads();
}

// Address resolution of one window, once at registration: every rank's copy + the multicast one.
__global__ void resolve_window_kernel(ncclDevComm dc, ncclWindow_t w, int P, char** out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (int p = 0; p < P; ++p) out[p] = static_cast<char*>(ncclGetPeerPointer(w, 0, p));
    out[P] = static_cast<char*>(ncclGetLsaMultimemPointer(w, 0, dc));
  }
}

// ------------------------------------------------------------------ copy-engine PS unit -----
// The data moves on the copy engines (cudaMemcpyAsync into the peers' windows: ~770 GB/s per
// direction at P = 2 on this pool against ~450 for SM-driven NVLink loads / stores, and no SMs
// taken from the co-running reconstructions); these kernels only signal, wait and apply.
// Receive window of a unit (symm_ce_bytes): [flag1: P u32 | pad][flag2: P u32 | pad] (4096 B),
// then P slots of S floats: slot p = rank p's piece of this rank's shard. Flags are reset-style
// (1 = arrived): each is reset by its consumer before the signal that lets the producer set it
// again, so a constant value works under CUDA-graph replay.
constexpr int64_t kCeHdr = 4096;

struct CeSignal {
  uint32_t* peer[kMaxPeers];   // flag[rank] in every peer's window (this rank's slot)
  uint32_t* reset;             // this rank's flag row to reset first (nullptr = none)
  int P, rank;
};

__global__ void ce_signal_kernel(CeSignal a) {
  const int t = threadIdx.x;
  if (a.reset) {
    if (t < a.P) a.reset[t] = 0u;
    __threadfence_system();
    __syncthreads();
  }
  if (t < a.P && t != a.rank) {
    __threadfence_system();   // the copies before this kernel in stream order are complete
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.peer[t]), "r"(1u) : "memory");
  }
}

// bounded wait for the P-1 peers' flags of a row, then reset them (the fresh shards are in W)
__global__ void ce_wait_kernel(uint32_t* flag, int P, int rank, unsigned long long timeout_ns,
                               int* err) {
  const int t = threadIdx.x;
  if (t < P && t != rank && poll_reached(flag + t, 1u, timeout_ns, err, kSiteCeShard)) flag[t] = 0u;
}

struct CeApply {
  const float* g;       // this rank's gradient, element 0 of the unit
  const float* recv;    // this rank's receive slots (slot p at p * S)
  float* W;             // this rank's W, element 0 of the unit
  uint32_t* flag;       // this rank's flag1 row
  int64_t S, lo, hi;
  int P, rank;
  float alpha;
  unsigned long long timeout_ns;
  int* err;
  KTrace trace, group;
};

// A7 on the owned shard once every peer's piece has arrived: W[lo+i] += alpha * sum_p piece_p[i],
// summed in rank order from piece 0 (the same arithmetic as the fused kernel's RANK_ORDER mode)
__global__ void __launch_bounds__(256) ce_apply_kernel(CeApply a) {
  ktrace_begin(a.trace);
  ktrace_begin(a.group);
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < a.P && threadIdx.x != a.rank &&
      !poll_reached(a.flag + threadIdx.x, 1u, a.timeout_ns, a.err, kSiteCeData))
    s_ok = 0;
  __syncthreads();
  if (s_ok) {
    const int64_t cnt = a.hi - a.lo, n4 = cnt / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    auto piece = [&](int p) { return p == a.rank ? a.g + a.lo : a.recv + (int64_t)p * a.S; };
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 s = reinterpret_cast<const float4*>(piece(0))[i];
      for (int p = 1; p < a.P; ++p) {
        const float4 t = reinterpret_cast<const float4*>(piece(p))[i];
        s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w;
      }
      float4* wp = reinterpret_cast<float4*>(a.W + a.lo) + i;
      float4 w = *wp;
      w.x = fmaf(a.alpha, s.x, w.x);
      w.y = fmaf(a.alpha, s.y, w.y);
      w.z = fmaf(a.alpha, s.z, w.z);
      w.w = fmaf(a.alpha, s.w, w.w);
      *wp = w;
    }
    if (blockIdx.x == 0)
      for (int64_t j = n4 * 4 + threadIdx.x; j < cnt; j += blockDim.x) {
        float s = piece(0)[j];
        for (int p = 1; p < a.P; ++p) s += piece(p)[j];
        a.W[a.lo + j] = fmaf(a.alpha, s, a.W[a.lo + j]);
      }
  }
  if (a.trace.rec || a.group.rec) {
    __syncthreads();
    ktrace_end(a.trace);
    ktrace_end(a.group);
  }
}

int grid_for(int64_t items, int threads, int cap) {
  int64_t g = (items + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// PS grid: a function of (n, P) only — the same on every rank (the last rank's shard may be short
// or empty; the kernel grid-strides over its own shard).
int ps_grid(pos_ctx* c, int64_t n, int P) {
  static const int ps_ctas_env = [] {
    const char* e = getenv("POS_NVLS_CTAS");
    return (e && *e) ? atoi(e) : 0;
  }();
  // NVLS loads have microsecond latency. Measured (VGG19-22K / VGG19 steps, next to the
  // reconstructions): P = 2 wants 64 CTAs (round 1: 0.45 -> 0.41 ms; 16: 0.52, 128: 0.47); P = 4
  // is best at 24-48 and 16 CTAs cost +17% (round 2: 0.363 vs 0.426 ms). Rule: 128 / P CTAs (the
  // same shard bytes per CTA), but >= 32 so a rank keeps enough NVLS loads in flight (P = 8: 32;
  // untested at P = 8 — the builder's boxes have at most 4 GPUs). P = 2 on the round-2 close
  // defaults (peer-load kernel, epoch barriers, pack placement): 96 CTAs beat 64 (VGG19 0.256 vs
  // 0.268 ms, VGG19-22K 0.337 vs 0.342; 128: VGG19 bimodal, 0.33 median).
  (void)c;
  int cap = ps_ctas_env > 0 ? ps_ctas_env : (P == 2 ? 96 : std::max(32, 128 / P));
  const int64_t S = pos_shard_stride(n, P);
  return grid_for(std::max<int64_t>(1, S / 4 / kPsUnroll), kPsThreads, cap);
}

// lane k: slot block at byte offset 256 k of the barrier window, epoch state at bar_state + 4 k
Xg make_xg(pos_ctx* c, int site, int lane = 0, uint32_t* exit_word = nullptr) {
  Xg x{};
  SymmState* st = state(c);
  if (st && st->bar.mc && c->world > 1) {
    x.mc = reinterpret_cast<uint32_t*>(st->bar.mc + kXgLaneBytes * lane);
    x.local = reinterpret_cast<uint32_t*>(st->bar.base + kXgLaneBytes * lane);
    x.state = st->bar_state + 4 * lane;
    x.exit_word = exit_word;
  }
  x.P = c->world;
  x.rank = c->rank;
  x.timeout_ns = c->timeout_ns;
  x.err = c->err_dev;
  x.site = site;
  return x;
}

Xg no_xg(pos_ctx* c) {
  Xg x{};
  x.P = c->world;
  x.timeout_ns = c->timeout_ns;
  x.err = c->err_dev;
  return x;
}

template <bool kRedMc, bool kStMc>
cudaError_t launch_ps(int grid, cudaStream_t s, PsArgs a, const Xg& x) {
  clear_stale_launch_error();
  if (a.trace.rec && a.trace.expected == 0) a.trace.expected = (unsigned)grid;
  ps_sync_kernel<kRedMc, kStMc><<<grid, kPsThreads, 0, s>>>(a, x);
  return cudaGetLastError();
}

template <bool kFlag, bool kMc>
cudaError_t launch_pack(int grid, cudaStream_t s, int32_t in_dtype, int32_t dtype,
                        const PackArgs& a, const Xg& x) {
  using bf = __nv_bfloat16;
  clear_stale_launch_error();
  if (dtype == POS_DT_BF16) {
    if (in_dtype == POS_IN_BF16) pack_x_kernel<bf, true, kFlag, kMc><<<grid, 256, 0, s>>>(a, x);
    else                         pack_x_kernel<float, true, kFlag, kMc><<<grid, 256, 0, s>>>(a, x);
  } else {
    if (in_dtype == POS_IN_BF16) pack_x_kernel<bf, false, kFlag, kMc><<<grid, 256, 0, s>>>(a, x);
    else                         pack_x_kernel<float, false, kFlag, kMc><<<grid, 256, 0, s>>>(a, x);
  }
  return cudaGetLastError();
}

int pack_grid(int64_t M, int64_t N, int64_t K, int32_t dtype) {
  static const int pack_ctas = [] {
    const char* e = getenv("POS_PACK_CTAS");
    const int v = (e && *e) ? atoi(e) : 128;
    return v < 1 ? 1 : v;
  }();
  const int vec = dtype == POS_DT_BF16 ? 8 : 4;
  return grid_for(K * rows_per_sample(dtype) * (row_elems(M, N) / vec), 256, pack_ctas);
}

}  // namespace

// ------------------------------------------------------------------------------- host --------
const char* site_name(int site) {
  switch (site) {
    case kSitePsEntry: return "PS unit entry barrier (a peer's gradients never arrived)";
    case kSitePsExit: return "PS unit exit barrier (a peer never finished its shard)";
    case kSitePackEntry: return "factor gather entry barrier";
    case kSitePackExit: return "factor gather exit barrier";
    case kSiteFlags: return "factor gather ready flags (a peer's slot never arrived)";
    case kSiteCeData: return "copy-engine PS: a peer's gradient piece never arrived";
    case kSiteCeShard: return "copy-engine PS: a peer's fresh shard never arrived";
    default: return "unknown cross-GPU wait";
  }
}

static int register_window(pos_ctx* c, SymmState* st, void* p, size_t bytes, SymmWindow* out) {
  ncclWindow_t win;
  ncclResult_t r = ncclCommWindowRegister(c->comm, p, bytes, &win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclCommWindowRegister");
  // NCCL's registration may leave a benign runtime error behind: consume it
  (void)cudaGetLastError();
  char** dtab = nullptr;
  POS_CUDA_TRY(cudaMalloc(&dtab, sizeof(char*) * (kMaxPeers + 1)));
  resolve_window_kernel<<<1, 32>>>(st->dev, win, c->world, dtab);
  cudaError_t e = cudaGetLastError();
  char* htab[kMaxPeers + 1] = {};
  if (e == cudaSuccess)
    e = cudaMemcpy(htab, dtab, sizeof(char*) * (c->world + 1), cudaMemcpyDeviceToHost);
  cudaFree(dtab);
  if (e != cudaSuccess) {
    ncclCommWindowDeregister(c->comm, win);
    return ctx_cuda_fail(c, e, "window address resolution");
  }
  out->base = static_cast<char*>(p);
  out->bytes = bytes;
  out->win = win;
  // peers through NCCL's flat LSA mapping; this rank through the allocation's own address (the
  // same physical memory — keeps local accesses on the regular mapping)
  for (int q = 0; q < c->world; ++q) out->peer[q] = q == c->rank ? out->base : htab[q];
  out->mc = htab[c->world];
  if (!out->mc || !htab[c->rank]) {
    ncclCommWindowDeregister(c->comm, win);
    POS_FAIL(POS_EUNSUPPORTED, "symmetric window without a multicast / peer mapping");
  }
  return POS_OK;
}

static int symm_init(pos_ctx* c) {
  if (c->symm) return POS_OK;
  POS_CHECK_ARG(c->comm, "symmetric memory needs a multi-rank context");
  POS_CHECK_ARG(c->world <= kMaxPeers, "symmetric memory supports at most %d ranks", kMaxPeers);
  SymmState* st = new SymmState();
  ncclDevCommRequirements reqs = {};
  reqs.lsaMultimem = true;
  ncclResult_t r = ncclDevCommCreate(c->comm, &reqs, &st->dev);
  if (r != ncclSuccess) {
    delete st;
    return ctx_nccl_fail(c, r, "ncclDevCommCreate(lsaMultimem)");
  }
  st->ready = true;
  if (st->dev.lsaSize != c->world || st->dev.lsaRank != c->rank) {
    ncclDevCommDestroy(c->comm, &st->dev);
    delete st;
    POS_FAIL(POS_EUNSUPPORTED, "the ranks do not form one NVLink (LSA) team");
  }
  // the cross-GPU barrier inboxes of the fused kernels
  void* p = nullptr;
  r = ncclMemAlloc(&p, 4096);
  if (r != ncclSuccess) {
    ncclDevCommDestroy(c->comm, &st->dev);
    delete st;
    return ctx_nccl_fail(c, r, "ncclMemAlloc(barrier)");
  }
  int rc = register_window(c, st, p, 4096, &st->bar);
  if (rc == POS_OK && (cudaMemset(p, 0, 4096) != cudaSuccess ||
                       cudaMalloc(&st->bar_state, 4 * kMaxLanes * sizeof(uint32_t)) != cudaSuccess ||
                       cudaMemset(st->bar_state, 0, 4 * kMaxLanes * sizeof(uint32_t)) != cudaSuccess ||
                       cudaDeviceSynchronize() != cudaSuccess))
    rc = ctx_cuda_fail(c, cudaGetLastError(), "barrier state");
  if (rc != POS_OK) {
    if (st->bar.win) ncclCommWindowDeregister(c->comm, st->bar.win);
    ncclMemFree(p);
    if (st->bar_state) cudaFree(st->bar_state);
    ncclDevCommDestroy(c->comm, &st->dev);
    delete st;
    return rc;
  }
  // with the collectives fused into our own kernels (which co-reside with the reconstruction
  // kernel) no SMs need to be kept free for NCCL CTAs
  if (!getenv("POS_SFB_MAX_CTAS")) c->max_ctas = 0;
  c->symm = st;
  return POS_OK;
}

void symm_destroy(pos_ctx* c) {
  SymmState* st = state(c);
  if (!st) return;
  for (auto& w : st->windows) {
    ncclCommWindowDeregister(c->comm, w.win);
    ncclMemFree(w.base);
  }
  if (st->bar.win) {
    ncclCommWindowDeregister(c->comm, st->bar.win);
    ncclMemFree(st->bar.base);
  }
  if (st->bar_state) cudaFree(st->bar_state);
  if (st->ready) ncclDevCommDestroy(c->comm, &st->dev);
  delete st;
  c->symm = nullptr;
}

static const SymmWindow* symm_find(pos_ctx* c, const void* p, size_t bytes, size_t* off) {
  SymmState* st = state(c);
  if (!st) return nullptr;
  const char* q = static_cast<const char*>(p);
  for (auto& w : st->windows)
    if (q >= w.base && q + bytes <= w.base + w.bytes) {
      *off = (size_t)(q - w.base);
      return &w;
    }
  return nullptr;
}

bool symm_lookup(pos_ctx* c, const void* p, size_t bytes) {
  size_t off;
  return symm_find(c, p, bytes, &off) != nullptr;
}

int symm_ps_grid(pos_ctx* c, int64_t n) { return ps_grid(c, n, c->world); }

int symm_ps_exit_wait(pos_ctx* c, const uint32_t* exit_word, int lane, cudaStream_t s) {
  SymmState* st = state(c);
  if (!st || !st->bar.mc || c->world < 2) return POS_OK;
  clear_stale_launch_error();
  xg_exit_wait_kernel<<<1, 32, 0, s>>>(
      reinterpret_cast<const uint32_t*>(st->bar.base + kXgLaneBytes * lane), exit_word, c->world,
      c->timeout_ns, c->err_dev, kSitePsExit);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "xg_exit_wait_kernel launch");
  return POS_OK;
}

int symm_ps_fused(pos_ctx* c, int64_t n, float* grad, float* W, float alpha, cudaStream_t s,
                  cudaEvent_t ev_a0, cudaEvent_t ev_a1, bool* done, KTrace tr, KTrace tg, int lane,
                  uint32_t* exit_word) {
  *done = false;
  const int P = c->world;
  if (P < 2 || c->local) return POS_OK;
  const int64_t padded = pos_padded_size(n, P);
  size_t og = 0, ow = 0;
  const SymmWindow* wg = symm_find(c, grad, (size_t)padded * 4, &og);
  const SymmWindow* ww = symm_find(c, W, (size_t)padded * 4, &ow);
  if (!wg || !ww || (og % 16) || (ow % 16)) return POS_OK;   // not symmetric: NCCL path
  PsArgs a{};
  a.g_mc = reinterpret_cast<const float*>(wg->mc + og);
  a.w_mc = reinterpret_cast<float*>(ww->mc + ow);
  for (int p = 0; p < P; ++p) {
    a.g[p] = reinterpret_cast<const float*>(wg->peer[p] + og);
    a.w[p] = reinterpret_cast<float*>(ww->peer[p] + ow);
  }
  a.wl = W;
  a.P = P;
  a.alpha = alpha;
  a.trace = tr;
  a.group = tg;
  pos_shard_range(n, P, c->rank, &a.lo, &a.hi);
  const Xg x = make_xg(c, kSitePsEntry, lane, exit_word);
  if (ev_a0) POS_CUDA_TRY(record_timing_event(ev_a0, s));
  const int grid = ps_grid(c, n, P);
  // P = 2: plain peer loads (summed in rank order: deterministic) + unicast peer stores move n/2 +
  // n/2 words per GPU and direction where the switch path moves ~1.5 n. Round 1 kept NVLS (the peer
  // path slowed a co-running reconstruction more); with the PS CTAs now co-resident with the
  // reconstruction and 64 MiB buckets, the peer path wins at P = 2 (round 2: VGG19-22K 0.426 ->
  // 0.338 ms, Inception-V3 0.296 -> 0.282 ms): POS_REDUCE_AUTO's choice at P = 2.
  cudaError_t e = cudaSuccess;
  if (c->fault == POS_FAULT_SKIP_PS && c->fault_rank == c->rank) {
    // fault injection: this rank never joins the unit (its peers' entry barriers time out)
  } else if (P == 2 && c->reduce_order == POS_REDUCE_AUTO) {
    e = launch_ps<false, false>(grid, s, a, x);   // rank-order peer loads, peer stores
  } else if (c->reduce_order == POS_REDUCE_RANK_ORDER) {
    e = launch_ps<false, true>(grid, s, a, x);   // deterministic sum, multicast broadcast
  } else {
    e = launch_ps<true, true>(grid, s, a, x);
  }
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "ps_sync_kernel launch");
  if (ev_a1) POS_CUDA_TRY(record_timing_event(ev_a1, s));
  *done = true;
  return POS_OK;
}

int64_t symm_ce_bytes(int64_t n, int P) { return kCeHdr + 4 * (int64_t)P * pos_shard_stride(n, P); }

int symm_ce_grid(pos_ctx* c, int64_t n) {
  int64_t lo = 0, hi = 0;
  pos_shard_range(n, c->world, c->rank, &lo, &hi);
  // at least one CTA: the apply kernel also consumes the peers' flags (an empty shard included)
  return std::max(1, ps_apply_grid(hi - lo));
}

int symm_ps_ce(pos_ctx* c, int64_t n, float* grad, float* W, void* ce_buf, float alpha,
               cudaStream_t s, cudaEvent_t ev_a0, cudaEvent_t ev_a1, bool* done, KTrace tr,
               KTrace tg) {
  *done = false;
  const int P = c->world, r = c->rank;
  if (P < 2 || c->local) return POS_OK;
  const int64_t S = pos_shard_stride(n, P);
  size_t ow = 0, oc = 0;
  const SymmWindow* ww = symm_find(c, W, (size_t)(S * P) * 4, &ow);
  const SymmWindow* wc = symm_find(c, ce_buf, (size_t)symm_ce_bytes(n, P), &oc);
  if (!ww || !wc) return POS_OK;
  if (ev_a0) POS_CUDA_TRY(record_timing_event(ev_a0, s));
  if (c->fault == POS_FAULT_SKIP_PS && c->fault_rank == r) {   // never joins: peers time out
    if (ev_a1) POS_CUDA_TRY(record_timing_event(ev_a1, s));
    *done = true;
    return POS_OK;
  }
  clear_stale_launch_error();
  auto flag_at = [&](int q, int row) {   // flag[row][r] in rank q's window
    return reinterpret_cast<uint32_t*>(wc->peer[q] + oc + 128 * row) + r;
  };
  // A6: push this rank's piece of every peer's shard into that peer's slot r
  for (int q = 0; q < P; ++q) {
    if (q == r) continue;
    int64_t lo = 0, hi = 0;
    pos_shard_range(n, P, q, &lo, &hi);
    if (hi > lo) {
      cudaError_t e = cudaMemcpyAsync(wc->peer[q] + oc + kCeHdr + 4 * (size_t)(r * S), grad + lo,
                                      4 * (size_t)(hi - lo), cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return ctx_cuda_fail(c, e, "copy-engine push (gradient piece)");
    }
  }
  CeSignal sg{};
  for (int q = 0; q < P; ++q) sg.peer[q] = flag_at(q, 0);
  sg.P = P;
  sg.rank = r;
  ce_signal_kernel<<<1, 32, 0, s>>>(sg);
  // A7: wait for the peers' pieces, sum in rank order, apply to the owned shard
  CeApply a{};
  a.g = grad;
  a.recv = reinterpret_cast<const float*>(wc->base + oc + kCeHdr);
  a.W = W;
  a.flag = reinterpret_cast<uint32_t*>(wc->base + oc);
  a.S = S;
  pos_shard_range(n, P, r, &a.lo, &a.hi);
  a.P = P;
  a.rank = r;
  a.alpha = alpha;
  a.timeout_ns = c->timeout_ns;
  a.err = c->err_dev;
  a.trace = tr;
  a.group = tg;
  const int grid = symm_ce_grid(c, n);
  if (a.trace.rec && a.trace.expected == 0) a.trace.expected = (unsigned)grid;
  ce_apply_kernel<<<grid, 256, 0, s>>>(a);
  if (ev_a1) POS_CUDA_TRY(record_timing_event(ev_a1, s));
  // A8: push the fresh shard into every replica, then signal (resetting this rank's flag1 row:
  // every apply CTA has consumed it) and wait for every peer's shard
  if (a.hi > a.lo)
    for (int q = 0; q < P; ++q) {
      if (q == r) continue;
      cudaError_t e = cudaMemcpyAsync(ww->peer[q] + ow + 4 * (size_t)a.lo, W + a.lo,
                                      4 * (size_t)(a.hi - a.lo), cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return ctx_cuda_fail(c, e, "copy-engine push (fresh shard)");
    }
  for (int q = 0; q < P; ++q) sg.peer[q] = flag_at(q, 1);
  sg.reset = a.flag;
  ce_signal_kernel<<<1, 32, 0, s>>>(sg);
  ce_wait_kernel<<<1, 32, 0, s>>>(reinterpret_cast<uint32_t*>(wc->base + oc + 128), P, r,
                                  c->timeout_ns, c->err_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "copy-engine PS kernels");
  *done = true;
  return POS_OK;
}

int symm_pack_mc(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                 const void* u, const void* v, void* gbuf, cudaStream_t s, bool* done,
                 void* gbuf2, uint32_t* flags, unsigned* fstate) {
  *done = false;
  if (c->world < 2 || c->local) return POS_OK;
  static const bool mc_off = [] {   // POS_PACK_MC=0: pack locally + NCCL all-gather instead
    const char* e = getenv("POS_PACK_MC");
    return e && e[0] == '0';
  }();
  if (mc_off) return POS_OK;
  const int P = c->world;
  const int64_t R = row_elems(M, N), eb = dtype_bytes(dtype);
  const size_t slot_bytes = (size_t)(K * rows_per_sample(dtype) * R * eb);
  size_t off = 0, off2 = 0, offf = 0;
  const SymmWindow* wb = symm_find(c, gbuf, slot_bytes * P, &off);
  if (!wb) return POS_OK;
  const bool flag_mode = gbuf2 && flags && fstate;
  const SymmWindow* wb2 = flag_mode ? symm_find(c, gbuf2, slot_bytes * P, &off2) : nullptr;
  const SymmWindow* wf = flag_mode ? symm_find(c, flags, sizeof(uint32_t) * P, &offf) : nullptr;
  if (flag_mode && (!wb2 || !wf)) return POS_OK;   // inconsistent registration: caller uses NCCL
  PackArgs a{};
  a.u = u; a.v = v;
  a.M = M; a.N = N; a.Mp = m_pad(M); a.R = R;
  a.K = K * rows_per_sample(dtype); a.Kp = K; a.split = rows_per_sample(dtype) == 3;
  a.P = P;
  const size_t mine = (size_t)c->rank * slot_bytes;
  a.mc[0] = wb->mc + off + mine;
  a.mc[1] = flag_mode ? wb2->mc + off2 + mine : a.mc[0];
  for (int p = 0; p < P; ++p) {
    a.dst[0][p] = wb->peer[p] + off + mine;
    a.dst[1][p] = flag_mode ? wb2->peer[p] + off2 + mine : a.dst[0][p];
  }
  if (flag_mode) {
    const size_t fo = offf + sizeof(uint32_t) * (size_t)c->rank;
    a.flag_mc = reinterpret_cast<uint32_t*>(wf->mc + fo);
    for (int p = 0; p < P; ++p) a.flag[p] = reinterpret_cast<uint32_t*>(wf->peer[p] + fo);
    a.state = fstate;
  }
  // POS_PACK_UC=1: P unicast stores through the peers' addresses instead of one multicast store
  static const bool uc = [] {
    const char* e = getenv("POS_PACK_UC");
    return e && e[0] == '1';
  }();
  const int grid = pack_grid(M, N, K, dtype);
  cudaError_t e;
  if (flag_mode) {
    e = uc ? launch_pack<true, false>(grid, s, in_dtype, dtype, a, no_xg(c))
           : launch_pack<true, true>(grid, s, in_dtype, dtype, a, no_xg(c));
  } else {
    e = launch_pack<false, true>(grid, s, in_dtype, dtype, a, make_xg(c, kSitePackEntry));
  }
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack_x_kernel launch");
  *done = true;
  return POS_OK;
}

int symm_wait_gathered(pos_ctx* c, const uint32_t* flags, const unsigned* fstate, int P,
                       cudaStream_t s) {
  clear_stale_launch_error();
  wait_flags_kernel<<<1, 32, 0, s>>>(flags, fstate, P, c->timeout_ns, c->err_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "wait_flags_kernel launch");
  return POS_OK;
}


cudaError_t preload_symm_kernels() {
  using bf = __nv_bfloat16;
  cudaFuncAttributes fa;
  const void* fns[] = {
      reinterpret_cast<const void*>(ps_sync_kernel<true, true>),
      reinterpret_cast<const void*>(ps_sync_kernel<false, true>),
      reinterpret_cast<const void*>(ps_sync_kernel<false, false>),
#define POS_PK(T, B, F, M) reinterpret_cast<const void*>(pack_x_kernel<T, B, F, M>)
      POS_PK(bf, true, true, true), POS_PK(bf, true, true, false), POS_PK(bf, true, false, true),
      POS_PK(bf, true, false, false), POS_PK(bf, false, true, true), POS_PK(bf, false, true, false),
      POS_PK(bf, false, false, true), POS_PK(bf, false, false, false), POS_PK(float, true, true, true),
      POS_PK(float, true, true, false), POS_PK(float, true, false, true), POS_PK(float, true, false, false),
      POS_PK(float, false, true, true), POS_PK(float, false, true, false), POS_PK(float, false, false, true),
      POS_PK(float, false, false, false),
#undef POS_PK
      reinterpret_cast<const void*>(wait_flags_kernel),
      reinterpret_cast<const void*>(xg_exit_wait_kernel),
      reinterpret_cast<const void*>(ce_signal_kernel),
      reinterpret_cast<const void*>(ce_wait_kernel),
      reinterpret_cast<const void*>(ce_apply_kernel),
      reinterpret_cast<const void*>(resolve_window_kernel)};
  for (const void* f : fns)
    if (cudaError_t e = cudaFuncGetAttributes(&fa, f); e != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace pos

using namespace pos;

// ----------------------------------------------------------------- single-GPU loopback ----
// P simulated ranks on one GPU, each with its own replica of the buffers; the P > 1 kernels above
// run for rank 0, 1, .., P-1 in stream order with pointer tables of the local replicas.
struct pos_loop_fc {
  pos_ctx* c = nullptr;
  int64_t M = 0, N = 0, K = 0;
  int32_t dtype = POS_DT_BF16;
  bool flag_mode = false;
  size_t slot_bytes = 0, buf_bytes = 0;   // one gather buffer = P slots
  std::vector<char*> buf;                 // per replica: [buffer 0 | buffer 1 | P flags] (flag mode)
  std::vector<unsigned*> gstate;          // per replica: gather state (2 x u32)
  std::vector<unsigned*> counter;         // per replica: dynamic tile scheduler state
  std::vector<SfbTcPlan> plan;
  std::vector<char> has_plan;
  std::vector<float*> W, b;
};

extern "C" {

int pos_mem_alloc(pos_ctx* c, int64_t bytes, void** out) {
  clear_error();
  POS_CHECK_ARG(c && out && bytes > 0, "bad arguments");
  int rc = symm_init(c);
  if (rc) return rc;
  void* p = nullptr;
  ncclResult_t r = ncclMemAlloc(&p, (size_t)bytes);
  if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclMemAlloc");
  SymmWindow w;
  if ((rc = register_window(c, state(c), p, (size_t)bytes, &w)) != POS_OK) {
    ncclMemFree(p);
    return rc;
  }
  state(c)->windows.push_back(w);
  cudaError_t e = cudaMemset(p, 0, (size_t)bytes);
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "cudaMemset(symmetric buffer)");
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "cudaDeviceSynchronize after pos_mem_alloc");
  *out = p;
  return POS_OK;
}

int pos_mem_free(pos_ctx* c, void* p) {
  clear_error();
  POS_CHECK_ARG(c && p, "bad arguments");
  SymmState* st = state(c);
  POS_CHECK_ARG(st, "no symmetric memory on this context");
  for (size_t i = 0; i < st->windows.size(); ++i)
    if (st->windows[i].base == p) {
      cudaDeviceSynchronize();
      ncclCommWindowDeregister(c->comm, st->windows[i].win);
      ncclMemFree(p);
      st->windows.erase(st->windows.begin() + i);
      return POS_OK;
    }
  POS_FAIL(POS_EINVAL, "pointer was not allocated by pos_mem_alloc");
}

int pos_mem_is_symmetric(pos_ctx* c, const void* p, int64_t bytes) {
  return (c && symm_lookup(c, p, (size_t)bytes)) ? 1 : 0;
}

int pos_loop_sync_layer_ps(pos_ctx* c, int64_t n, float* const* grads, float* const* W,
                           float alpha, void* stream) {
  clear_error();
  POS_CHECK_ARG(c && c->local, "pos_loop_* needs a context from pos_init_local");
  POS_CHECK_ARG(n >= 1 && grads && W, "bad arguments");
  const int P = c->world;
  POS_CHECK_ARG(P <= kMaxPeers, "at most %d loopback ranks", kMaxPeers);
  for (int p = 0; p < P; ++p)
    POS_CHECK_ARG(grads[p] && W[p] && aligned16(grads[p]) && aligned16(W[p]),
                  "rank %d: grad and W must be non-NULL and 16-byte aligned", p);
  int rc = ctx_check(c);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  PsArgs a{};
  for (int p = 0; p < P; ++p) {
    a.g[p] = grads[p];
    a.w[p] = W[p];
  }
  a.P = P;
  a.alpha = alpha;
  const int grid = ps_grid(c, n, P);
  for (int r = 0; r < P; ++r) {   // every rank's fused reduce + apply + broadcast of its shard
    pos_shard_range(n, P, r, &a.lo, &a.hi);
    a.wl = W[r];
    cudaError_t e = launch_ps<false, false>(grid, s, a, no_xg(c));
    if (e != cudaSuccess) return ctx_cuda_fail(c, e, "ps_sync_kernel launch (loopback)");
  }
  return POS_OK;
}

int pos_loop_sync_layer_ps_ce(pos_ctx* c, int64_t n, float* const* grads, float* const* W,
                              float alpha, void* stream) {
  clear_error();
  POS_CHECK_ARG(c && c->local, "pos_loop_* needs a context from pos_init_local");
  POS_CHECK_ARG(n >= 1 && grads && W, "bad arguments");
  const int P = c->world;
  POS_CHECK_ARG(P <= kMaxPeers, "at most %d loopback ranks", kMaxPeers);
  for (int p = 0; p < P; ++p)
    POS_CHECK_ARG(grads[p] && W[p] && aligned16(grads[p]) && aligned16(W[p]),
                  "rank %d: grad and W must be non-NULL and 16-byte aligned", p);
  int rc = ctx_check(c);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t S = pos_shard_stride(n, P);
  const size_t bytes = (size_t)symm_ce_bytes(n, P);   // one replica's receive window
  void* ws = nullptr;
  if ((rc = ctx_workspace(c, bytes * P, &ws))) return rc;
  std::vector<char*> rb(P);
  for (int p = 0; p < P; ++p) {
    rb[p] = static_cast<char*>(ws) + bytes * p;
    POS_CUDA_TRY(cudaMemsetAsync(rb[p], 0, kCeHdr, s));   // flags (the workspace is shared)
  }
  auto flag = [&](int q, int row, int r) { return reinterpret_cast<uint32_t*>(rb[q] + 128 * row) + r; };
  clear_stale_launch_error();
  // The copy-engine PS unit of every rank, phase by phase (a rank's apply waits for every peer's
  // push, so the ranks cannot simply run one after the other): pushes + signals, applies, shard
  // pushes + signals, completion waits — the kernels and copies symm_ps_ce issues per rank.
  for (int r = 0; r < P; ++r) {
    CeSignal sg{};
    for (int q = 0; q < P; ++q) {
      sg.peer[q] = flag(q, 0, r);
      int64_t lo = 0, hi = 0;
      pos_shard_range(n, P, q, &lo, &hi);
      if (q != r && hi > lo)
        POS_CUDA_TRY(cudaMemcpyAsync(rb[q] + kCeHdr + 4 * (size_t)(r * S), grads[r] + lo,
                                     4 * (size_t)(hi - lo), cudaMemcpyDeviceToDevice, s));
    }
    sg.P = P;
    sg.rank = r;
    ce_signal_kernel<<<1, 32, 0, s>>>(sg);
  }
  for (int r = 0; r < P; ++r) {
    CeApply a{};
    a.g = grads[r];
    a.recv = reinterpret_cast<const float*>(rb[r] + kCeHdr);
    a.W = W[r];
    a.flag = flag(r, 0, 0);
    a.S = S;
    pos_shard_range(n, P, r, &a.lo, &a.hi);
    a.P = P;
    a.rank = r;
    a.alpha = alpha;
    a.timeout_ns = c->timeout_ns;
    a.err = c->err_dev;
    ce_apply_kernel<<<std::max(1, ps_apply_grid(a.hi - a.lo)), 256, 0, s>>>(a);
  }
  for (int r = 0; r < P; ++r) {
    int64_t lo = 0, hi = 0;
    pos_shard_range(n, P, r, &lo, &hi);
    CeSignal sg{};
    for (int q = 0; q < P; ++q) {
      sg.peer[q] = flag(q, 1, r);
      if (q != r && hi > lo)
        POS_CUDA_TRY(cudaMemcpyAsync(W[q] + lo, W[r] + lo, 4 * (size_t)(hi - lo),
                                     cudaMemcpyDeviceToDevice, s));
    }
    sg.reset = flag(r, 0, 0);
    sg.P = P;
    sg.rank = r;
    ce_signal_kernel<<<1, 32, 0, s>>>(sg);
  }
  for (int r = 0; r < P; ++r)
    ce_wait_kernel<<<1, 32, 0, s>>>(flag(r, 1, 0), P, r, c->timeout_ns, c->err_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "copy-engine PS kernels (loopback)");
  return POS_OK;
}

int pos_loop_fc_create(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t dtype,
                       float* const* W, float* const* b, pos_loop_fc** out) {
  clear_error();
  POS_CHECK_ARG(c && c->local && out, "pos_loop_* needs a context from pos_init_local");
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && M <= (1LL << 31) && N <= (1LL << 31), "bad M, N, K");
  POS_CHECK_ARG(dtype == POS_DT_BF16 || dtype == POS_DT_TF32 || dtype == POS_DT_F32, "bad dtype");
  const int P = c->world;
  POS_CHECK_ARG(P <= kMaxPeers, "at most %d loopback ranks", kMaxPeers);
  POS_CHECK_ARG(W, "NULL W table");
  const bool fm = gather_flag_mode(dtype, N);
  for (int p = 0; p < P; ++p) {
    POS_CHECK_ARG(W[p], "rank %d: NULL W", p);
    POS_CHECK_ARG(!fm || aligned16(W[p]), "rank %d: W must be 16-byte aligned", p);
  }
  pos_loop_fc* lf = new pos_loop_fc();
  lf->c = c;
  lf->M = M; lf->N = N; lf->K = K;
  lf->dtype = dtype;
  lf->flag_mode = fm;
  lf->slot_bytes = (size_t)(K * rows_per_sample(dtype) * row_elems(M, N) * dtype_bytes(dtype));
  lf->buf_bytes = (lf->slot_bytes * P + 255) & ~size_t(255);
  const size_t alloc = fm ? 2 * lf->buf_bytes + 256 : lf->buf_bytes;
  lf->buf.assign(P, nullptr);
  lf->gstate.assign(P, nullptr);
  lf->counter.assign(P, nullptr);
  lf->plan.resize(P);
  lf->has_plan.assign(P, 0);
  lf->W.assign(W, W + P);
  lf->b.assign(P, nullptr);
  if (b)
    for (int p = 0; p < P; ++p) lf->b[p] = b[p];
  int rc = POS_OK;
  for (int p = 0; p < P && rc == POS_OK; ++p) {
    if (cudaMalloc(&lf->buf[p], alloc) != cudaSuccess ||
        cudaMemset(lf->buf[p], 0, alloc) != cudaSuccess ||
        cudaMalloc(&lf->gstate[p], 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(lf->gstate[p], 0, 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMalloc(&lf->counter[p], 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(lf->counter[p], 0, 2 * sizeof(unsigned)) != cudaSuccess) {
      (void)cudaGetLastError();
      rc = POS_ENOMEM;
      set_error("loopback buffers: cudaMalloc failed");
      break;
    }
    if (fm) {
      SfbTcPlan& pl = lf->plan[p];
      lf->has_plan[p] = sfb_tc_make_plan(&pl, M, N, K * P, dtype, lf->buf[p], W[p], N,
                                         c->max_ctas, lf->b[p], lf->buf[p] + lf->buf_bytes);
      if (!lf->has_plan[p]) {
        rc = POS_EUNSUPPORTED;
        set_error("flag-mode gather without a tensor-core plan");
        break;
      }
      pl.counter = lf->counter[p];
      pl.gsel = lf->gstate[p];
    }
  }
  if (rc != POS_OK) {
    pos_loop_fc_destroy(lf);
    return rc;
  }
  *out = lf;
  return POS_OK;
}

int pos_loop_fc_sync(pos_loop_fc* lf, int32_t in_dtype, const void* const* u,
                     const void* const* v, float alpha, void* stream) {
  clear_error();
  POS_CHECK_ARG(lf && u && v, "bad arguments");
  POS_CHECK_ARG(in_dtype == POS_IN_BF16 || in_dtype == POS_IN_F32, "bad in_dtype");
  pos_ctx* c = lf->c;
  const int P = c->world;
  for (int p = 0; p < P; ++p) POS_CHECK_ARG(u[p] && v[p], "rank %d: NULL factors", p);
  int rc = ctx_check(c);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  // A2 + A3: every rank packs its factors into its slot of every replica's gather buffer
  PackArgs a{};
  a.M = lf->M; a.N = lf->N; a.Mp = m_pad(lf->M); a.R = row_elems(lf->M, lf->N);
  a.K = lf->K * rows_per_sample(lf->dtype); a.Kp = lf->K; a.split = rows_per_sample(lf->dtype) == 3;
  a.P = P;
  const int grid = pack_grid(lf->M, lf->N, lf->K, lf->dtype);
  for (int r = 0; r < P; ++r) {
    if (c->fault == POS_FAULT_SKIP_PACK && c->fault_rank == r) continue;   // fault injection
    a.u = u[r];
    a.v = v[r];
    const size_t mine = (size_t)r * lf->slot_bytes;
    for (int p = 0; p < P; ++p) {
      a.dst[0][p] = lf->buf[p] + mine;
      a.dst[1][p] = lf->flag_mode ? lf->buf[p] + lf->buf_bytes + mine : a.dst[0][p];
      a.flag[p] = lf->flag_mode
                      ? reinterpret_cast<uint32_t*>(lf->buf[p] + 2 * lf->buf_bytes) + r
                      : nullptr;
    }
    a.state = lf->gstate[r];
    cudaError_t e = lf->flag_mode
                        ? launch_pack<true, false>(grid, s, in_dtype, lf->dtype, a, no_xg(c))
                        : launch_pack<false, false>(grid, s, in_dtype, lf->dtype, a, no_xg(c));
    if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack_x_kernel launch (loopback)");
  }
  // A4 + A4b on every replica, each behind its own ready-flag wait
  for (int r = 0; r < P; ++r) {
    if (lf->flag_mode) {
      const uint32_t* flags = reinterpret_cast<const uint32_t*>(lf->buf[r] + 2 * lf->buf_bytes);
      if ((rc = symm_wait_gathered(c, flags, lf->gstate[r], P, s))) return rc;
      cudaError_t e = sfb_tc_launch(lf->plan[r], alpha, 1, s);
      if (e != cudaSuccess) return ctx_cuda_fail(c, e, "reconstruct launch (loopback)");
    } else {
      rc = reconstruct_apply(lf->M, lf->N, lf->K * P, lf->dtype, lf->buf[r], 1, lf->W[r], lf->N,
                             lf->b[r], alpha, c->max_ctas, s);
      if (rc != POS_OK) { if (c->sticky == POS_OK) c->sticky = rc; return rc; }
    }
  }
  return POS_OK;
}

int pos_loop_fc_destroy(pos_loop_fc* lf) {
  clear_error();
  if (!lf) return POS_OK;
  cudaDeviceSynchronize();
  for (char* p : lf->buf) if (p) cudaFree(p);
  for (unsigned* p : lf->gstate) if (p) cudaFree(p);
  for (unsigned* p : lf->counter) if (p) cudaFree(p);
  delete lf;
  return POS_OK;
}

}  // extern "C"
