// NVLink-SHARP / symmetric-memory path: the PS and SFB collectives fused into
// the kernels that consume them, over NVSwitch multicast (NVLS) memory registered as NCCL symmetric
// windows. NCCL provides only the plumbing (allocation, window registration, the device-side
// pointers and the cross-GPU barrier); the data movement and arithmetic are these kernels.
//
//  * ps_nvls_kernel (A6 + A7 + A8 fused): rank r owns shard [lo, hi) of a dense unit.
//      ghat = multimem.ld_reduce.add(grad[i])      -- the switch sums all P workers' gradients
//      w    = W_local[i] + alpha * ghat            -- the server's "apply (+)"
//      multimem.st(W[i], w)                        -- fresh parameters to every replica
//    bracketed by two LSA barriers: gradients of all ranks complete before the reduce, every
//    replica's W complete (and every gradient consumed) before any rank proceeds.
//  * pack_mc_kernel (A2 + A3 fused): this rank's sufficient factors, packed and cast,
//    are multicast-stored into its slot of EVERY rank's gather buffer (one NVLink egress copy; the
//    switch replicates), followed by an LSA barrier so the reconstruction can read all P slots.
//
// All fused kernels of a context run on its comm stream, in the same order on every rank, so one
// set of barrier indices [0, kBarriers) is reused sequentially (the session epochs persist in the
// barrier resource buffer, also across CUDA-graph replays).
#include <cuda_bf16.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdlib>
#include <vector>

#include "ctx.h"

namespace pos {

constexpr int kBarriers = 128;  // max CTAs of a fused kernel

struct SymmWindow {
  char* base;
  size_t bytes;
  ncclWindow_t win;
};

struct SymmState {
  ncclDevComm dev;
  bool ready = false;
  bool multimem = false;
  std::vector<SymmWindow> windows;
};

static SymmState* state(pos_ctx* c) { return static_cast<SymmState*>(c->symm); }

namespace {

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

#ifndef POS_PACK_CTA_FENCE
#define POS_PACK_CTA_FENCE 1
#endif
#ifndef POS_ENTRY_ORDER
#define POS_ENTRY_ORDER cuda::memory_order_acquire
#endif
constexpr cuda::memory_order kEntryOrder = POS_ENTRY_ORDER;

constexpr int kPsThreads = 512;
#ifndef POS_NVLS_UNROLL
#define POS_NVLS_UNROLL 4
#endif
constexpr int kPsUnroll = POS_NVLS_UNROLL;   // 16-byte NVLS reductions in flight per thread

__global__ void __launch_bounds__(kPsThreads)
ps_nvls_kernel(ncclDevComm dc, ncclWindow_t wg, size_t off_g, ncclWindow_t ww, size_t off_w,
               int64_t lo, int64_t hi, float alpha) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, true);
  // Entry: every worker's gradient is in place. The gradients were written by kernels that have
  // completed (stream order), i.e. they are in each GPU's L2, where NVLS reads are served: the
  // arrival needs no release fence (POS_ENTRY_ORDER selects the order for experiments).
  bar.sync(ncclCoopCta(), kEntryOrder);
  const float* gmc = static_cast<const float*>(ncclGetLsaMultimemPointer(wg, off_g, dc));
  float* wmc = static_cast<float*>(ncclGetLsaMultimemPointer(ww, off_w, dc));
  const float* wl = static_cast<const float*>(ncclGetLocalPointer(ww, off_w));
  const int64_t v0 = lo / 4, v1 = hi / 4;   // lo is a multiple of 64
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = v0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kPsUnroll - 1) * stride < v1; i += kPsUnroll * stride) {
    float4 g[kPsUnroll], w[kPsUnroll];
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      g[u] = mm_ld_reduce_v4(gmc + 4 * (i + u * stride));
      w[u] = *reinterpret_cast<const float4*>(wl + 4 * (i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      w[u].x = fmaf(alpha, g[u].x, w[u].x);
      w[u].y = fmaf(alpha, g[u].y, w[u].y);
      w[u].z = fmaf(alpha, g[u].z, w[u].z);
      w[u].w = fmaf(alpha, g[u].w, w[u].w);
      mm_st_v4(wmc + 4 * (i + u * stride), w[u]);
    }
  }
  for (; i < v1; i += stride) {
    float4 g = mm_ld_reduce_v4(gmc + 4 * i);
    float4 w = *reinterpret_cast<const float4*>(wl + 4 * i);
    w.x = fmaf(alpha, g.x, w.x);
    w.y = fmaf(alpha, g.y, w.y);
    w.z = fmaf(alpha, g.z, w.z);
    w.w = fmaf(alpha, g.w, w.w);
    mm_st_v4(wmc + 4 * i, w);
  }
  if (blockIdx.x == 0)   // scalar tail of the shard
    for (int64_t j = v1 * 4 + threadIdx.x; j < hi; j += blockDim.x)
      mm_st(wmc + j, fmaf(alpha, mm_ld_reduce(gmc + j), wl[j]));
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);   // every replica's W is complete
}

// P = 2 variant of the fused PS step with plain peer loads / stores over NVLink (LSA pointers):
// per GPU and direction it moves n/2 + n/2 fp32 words where the NVLS path moves ~1.5 n (the switch
// reads every copy, including the local one, and writes every replica). Sum in rank order.
__global__ void __launch_bounds__(kPsThreads)
ps_p2p2_kernel(ncclDevComm dc, ncclWindow_t wg, size_t off_g, ncclWindow_t ww, size_t off_w,
               int64_t lo, int64_t hi, float alpha) {
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, true);
  bar.sync(ncclCoopCta(), kEntryOrder);     // both gradients are in place (see ps_nvls_kernel)
  const float* g0 = static_cast<const float*>(ncclGetLsaPointer(wg, off_g, 0));
  const float* g1 = static_cast<const float*>(ncclGetLsaPointer(wg, off_g, 1));
  float* w0 = static_cast<float*>(ncclGetLsaPointer(ww, off_w, 0));
  float* w1 = static_cast<float*>(ncclGetLsaPointer(ww, off_w, 1));
  const float* wl = static_cast<const float*>(ncclGetLocalPointer(ww, off_w));
  const int64_t v0 = lo / 4, v1 = hi / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = v0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kPsUnroll - 1) * stride < v1; i += kPsUnroll * stride) {
    float4 a[kPsUnroll], b[kPsUnroll], w[kPsUnroll];
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      a[u] = *reinterpret_cast<const float4*>(g0 + 4 * (i + u * stride));
      b[u] = *reinterpret_cast<const float4*>(g1 + 4 * (i + u * stride));
      w[u] = *reinterpret_cast<const float4*>(wl + 4 * (i + u * stride));
    }
#pragma unroll
    for (int u = 0; u < kPsUnroll; ++u) {
      w[u].x = fmaf(alpha, a[u].x + b[u].x, w[u].x);
      w[u].y = fmaf(alpha, a[u].y + b[u].y, w[u].y);
      w[u].z = fmaf(alpha, a[u].z + b[u].z, w[u].z);
      w[u].w = fmaf(alpha, a[u].w + b[u].w, w[u].w);
      *reinterpret_cast<float4*>(w0 + 4 * (i + u * stride)) = w[u];
      *reinterpret_cast<float4*>(w1 + 4 * (i + u * stride)) = w[u];
    }
  }
  for (; i < v1; i += stride) {
    const float4 a = *reinterpret_cast<const float4*>(g0 + 4 * i);
    const float4 b = *reinterpret_cast<const float4*>(g1 + 4 * i);
    float4 w = *reinterpret_cast<const float4*>(wl + 4 * i);
    w.x = fmaf(alpha, a.x + b.x, w.x);
    w.y = fmaf(alpha, a.y + b.y, w.y);
    w.z = fmaf(alpha, a.z + b.z, w.z);
    w.w = fmaf(alpha, a.w + b.w, w.w);
    *reinterpret_cast<float4*>(w0 + 4 * i) = w;
    *reinterpret_cast<float4*>(w1 + 4 * i) = w;
  }
  if (blockIdx.x == 0)   // scalar tail of the shard
    for (int64_t j = v1 * 4 + threadIdx.x; j < hi; j += blockDim.x) {
      const float w = fmaf(alpha, g0[j] + g1[j], wl[j]);
      w0[j] = w;
      w1[j] = w;
    }
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);   // both replicas of W are complete
}

__device__ __forceinline__ float ld_in(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_in(const float* p) { return *p; }

// Gather state of one SFB unit in flag mode (device memory of this rank, zero-initialised):
// [0] packs completed by this rank (= iteration sequence), [1] CTAs of the running pack done.
struct GatherFlags {
  ncclWindow_t win;      // symmetric window holding the unit's P ready flags
  size_t off_mine;       // offset of flag[rank] (written by this rank into every replica)
  unsigned* state;       // this rank's GatherFlags state (2 x u32)
};

// One 16-byte output vector per thread iteration, multicast to every rank's gather buffer.
//  kFlag = false: barrier mode — an entry barrier (cross-rank WAR on the single gather buffer) and
//    an exit barrier (all P slots have landed everywhere) around the multicast.
//  kFlag = true: flag mode — no waiting at all: the gather buffer is double-buffered by the
//    iteration parity read from device memory (so a replayed CUDA graph alternates too), and the
//    last CTA to finish publishes "slot of rank r for iteration s is complete" as a release-store
//    of s into flag[r] of every replica. The consumer waits for the P flags (wait_flags_kernel).
//    WAR safety: rank r writes buffer s%2 at iteration s only after its iteration s-1 consumed
//    every rank's s-1 flag, and each rank publishes its s-1 flag only after finishing iteration
//    s-2, whose reconstruction was the last reader of buffer s%2.
//  kUC (flag mode only): P unicast stores through the peers' LSA pointers instead of one
//    multimem store (an experiment knob, POS_PACK_UC=1).
template <typename Tin, bool kBF16, bool kFlag, bool kUC = false>
__global__ void __launch_bounds__(256)
pack_mc_kernel(ncclDevComm dc, ncclWindow_t wgb, size_t off_slot, size_t off_slot2,
               const Tin* __restrict__ u, const Tin* __restrict__ v, int64_t M, int64_t N,
               int64_t Mp, int64_t R, int64_t K, GatherFlags gf, int P = 0) {
  uint32_t seq = 0;
  if constexpr (!kFlag) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, true);
    // Entry barrier: every rank has reached this iteration's pack on its comm stream, which (by
    // pos_sched_end's contract) is after its previous reconstruction finished reading the gather
    // buffer we are about to overwrite (cross-rank WAR).
    bar.sync(ncclCoopCta(), kEntryOrder);
  } else {
    seq = *reinterpret_cast<volatile unsigned*>(gf.state);
  }
  const size_t off = (kFlag && (seq & 1)) ? off_slot2 : off_slot;
  float* dst = kUC ? nullptr : static_cast<float*>(ncclGetLsaMultimemPointer(wgb, off, dc));
  float* peer_dst[8];
  if constexpr (kUC)
    for (int p = 0; p < P && p < 8; ++p) peer_dst[p] = static_cast<float*>(ncclGetLsaPointer(wgb, off, p));
  constexpr int VEC = kBF16 ? 8 : 4;
  const int64_t chunks_per_row = R / VEC, total = K * chunks_per_row;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < total;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = c / chunks_per_row, col = (c % chunks_per_row) * VEC;
    const Tin* src;
    int64_t idx, lim;
    if (col < Mp) { src = u + k * M; idx = col; lim = M; }
    else          { src = v + k * N; idx = col - Mp; lim = N; }
    const int64_t onec = col < Mp ? -1 : N;   // ones column (fused bias), as in pack_*_kernel
    float4 o;
    if constexpr (kBF16) {
      __align__(16) __nv_bfloat16 h[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        h[i] = __float2bfloat16_rn(idx + i < lim ? ld_in(src + idx + i) : (idx + i == onec ? 1.f : 0.f));
      o = *reinterpret_cast<const float4*>(h);   // bit pattern only; a store does not convert
    } else {
      o.x = idx + 0 < lim ? ld_in(src + idx + 0) : (idx + 0 == onec ? 1.f : 0.f);
      o.y = idx + 1 < lim ? ld_in(src + idx + 1) : (idx + 1 == onec ? 1.f : 0.f);
      o.z = idx + 2 < lim ? ld_in(src + idx + 2) : (idx + 2 == onec ? 1.f : 0.f);
      o.w = idx + 3 < lim ? ld_in(src + idx + 3) : (idx + 3 == onec ? 1.f : 0.f);
    }
    // element offset of this 16-byte vector in float units: (k * R + col) * eb / 4
    const int64_t eo = ((k * R + col) * (kBF16 ? 2 : 4)) / 4;
    if constexpr (kUC) {
      for (int p = 0; p < P && p < 8; ++p) *reinterpret_cast<float4*>(peer_dst[p] + eo) = o;
    } else {
      mm_st_v4(dst + eo, o);
    }
  }
  if constexpr (!kFlag) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, true);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);   // all P slots have landed everywhere
  } else {
#if POS_PACK_CTA_FENCE
    __syncthreads();                        // the CTA's stores happen-before thread 0's fence
    if (threadIdx.x == 0) __threadfence_system();
#else
    __threadfence_system();                 // this thread's multicast stores are performed
    __syncthreads();
#endif
    if (threadIdx.x == 0) {
      const unsigned prev = atomicAdd(gf.state + 1, 1u);
      if (prev == gridDim.x - 1) {          // last CTA: every CTA's stores are performed
        __threadfence_system();
        gf.state[1] = 0;
        gf.state[0] = seq + 1;
        if constexpr (kUC) {
          for (int p = 0; p < P && p < 8; ++p) {
            uint32_t* f = static_cast<uint32_t*>(ncclGetLsaPointer(gf.win, gf.off_mine, p));
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(seq + 1) : "memory");
          }
        } else {
          uint32_t* fmc =
              static_cast<uint32_t*>(ncclGetLsaMultimemPointer(gf.win, gf.off_mine, dc));
          asm volatile("multimem.st.release.sys.global.u32 [%0], %1;" ::"l"(fmc), "r"(seq + 1)
                       : "memory");
        }
      }
    }
  }
}

// Consumer side of flag mode: returns once every rank's slot of this iteration is in place
// (flag[r] >= this rank's own sequence, which its pack has just advanced).
__global__ void wait_flags_kernel(const uint32_t* flags, const unsigned* state, int P) {
  const uint32_t want = *reinterpret_cast<const volatile unsigned*>(state);
  for (int r = threadIdx.x; r < P; r += blockDim.x) {
    uint32_t got;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(got) : "l"(flags + r) : "memory");
    } while ((int32_t)(got - want) < 0);
  }
  __syncthreads();
}

int grid_for(int64_t items, int threads, int cap) {
  int64_t g = (items + threads - 1) / threads;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

// ------------------------------------------------------------------------------- host --------
static int symm_init(pos_ctx* c) {
  if (c->symm) return POS_OK;
  POS_CHECK_ARG(c->comm, "symmetric memory needs a multi-rank context");
  SymmState* st = new SymmState();
  ncclDevCommRequirements reqs = {};
  reqs.lsaMultimem = true;
  reqs.lsaBarrierCount = kBarriers;
  ncclResult_t r = ncclDevCommCreate(c->comm, &reqs, &st->dev);
  if (r != ncclSuccess) {
    delete st;
    return ctx_nccl_fail(c, r, "ncclDevCommCreate(lsaMultimem)");
  }
  st->ready = true;
  // with the collectives fused into our own kernels (which co-reside with the reconstruction
  // kernel) no SMs need to be kept free for NCCL CTAs
  if (!getenv("POS_SFB_MAX_CTAS")) c->max_ctas = 0;
  st->multimem = true;
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
  if (st->ready) ncclDevCommDestroy(c->comm, &st->dev);
  delete st;
  c->symm = nullptr;
}

bool symm_lookup(pos_ctx* c, const void* p, size_t bytes, ncclWindow_t* win, size_t* off) {
  SymmState* st = state(c);
  if (!st || !st->multimem) return false;
  const char* q = static_cast<const char*>(p);
  for (auto& w : st->windows)
    if (q >= w.base && q + bytes <= w.base + w.bytes) {
      *win = w.win;
      *off = (size_t)(q - w.base);
      return true;
    }
  return false;
}

int symm_ps_fused(pos_ctx* c, int64_t n, float* grad, float* W, float alpha, cudaStream_t s,
                  cudaEvent_t ev_a0, cudaEvent_t ev_a1, bool* done) {
  clear_stale_launch_error();
  *done = false;
  const int P = c->world;
  if (P < 2 || c->local) return POS_OK;
  const int64_t padded = pos_padded_size(n, P);
  ncclWindow_t wg, ww;
  size_t og, ow;
  if (!symm_lookup(c, grad, (size_t)padded * 4, &wg, &og) ||
      !symm_lookup(c, W, (size_t)padded * 4, &ww, &ow) || (og % 16) || (ow % 16))
    return POS_OK;   // not symmetric: caller uses the NCCL path
  int64_t lo = 0, hi = 0;
  pos_shard_range(n, P, c->rank, &lo, &hi);
  if (ev_a0) POS_CUDA_TRY(record_timing_event(ev_a0, s));
  // NVLS loads have microsecond latency. Measured (VGG19-22K / VGG19 steps, next to the
  // reconstructions): P = 2 — each rank reduces half of every unit — wants 64 CTAs (0.45 -> 0.41 ms;
  // 16: 0.52, 128: 0.47); P = 4 is best at 24-48 (64 hung once at P = 4: NVLS CTAs spinning in
  // their barrier can starve the reconstructions and packs of SM slots). Rule: 128 / P CTAs (the
  // same shard bytes per CTA at every P), at least 16 — P = 8 (not measurable here) gets 16.
  static const int ps_ctas_env = [] {
    const char* e = getenv("POS_NVLS_CTAS");
    return (e && *e) ? atoi(e) : 0;
  }();
  int ps_ctas = ps_ctas_env > 0 ? ps_ctas_env : std::max(16, 128 / P);
  if (ps_ctas > kBarriers) ps_ctas = kBarriers;
  const int grid = grid_for(std::max<int64_t>(1, (hi - lo) / 4 / kPsUnroll), kPsThreads, ps_ctas);
  // P = 2 option (POS_PS_P2P=1): plain peer loads / stores move less over NVLink than the switch
  // path — 10-20% faster alone (80 MB: 196 vs 218 us), but its NVLink traffic through the SMs'
  // load/store path slows a concurrent reconstruction far more (VGG19-22K step 0.55 vs 0.45 ms);
  // only the PS-only Inception-V3 step gains (-8%), so the NVLS kernel stays the default
  static const bool p2p2 = [] {
    const char* e = getenv("POS_PS_P2P");
    return e && e[0] == '1';
  }();
  if (P == 2 && p2p2)
    ps_p2p2_kernel<<<grid, kPsThreads, 0, s>>>(state(c)->dev, wg, og, ww, ow, lo, hi, alpha);
  else
    ps_nvls_kernel<<<grid, kPsThreads, 0, s>>>(state(c)->dev, wg, og, ww, ow, lo, hi, alpha);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "ps_nvls_kernel launch");
  if (ev_a1) POS_CUDA_TRY(record_timing_event(ev_a1, s));
  *done = true;
  return POS_OK;
}

namespace {
template <bool kFlag, bool kUC = false>
void launch_pack_mc(int grid, cudaStream_t s, const ncclDevComm& dc, ncclWindow_t wgb,
                    size_t off_slot, size_t off_slot2, int32_t in_dtype, int32_t dtype,
                    const void* u, const void* v, int64_t M, int64_t N, int64_t Mp, int64_t R,
                    int64_t K, GatherFlags gf, int P = 0) {
  using bf = __nv_bfloat16;
  if (dtype == POS_DT_BF16) {
    if (in_dtype == POS_IN_BF16)
      pack_mc_kernel<bf, true, kFlag, kUC><<<grid, 256, 0, s>>>(
          dc, wgb, off_slot, off_slot2, static_cast<const bf*>(u), static_cast<const bf*>(v), M, N,
          Mp, R, K, gf, P);
    else
      pack_mc_kernel<float, true, kFlag, kUC><<<grid, 256, 0, s>>>(
          dc, wgb, off_slot, off_slot2, static_cast<const float*>(u),
          static_cast<const float*>(v), M, N, Mp, R, K, gf, P);
  } else {
    if (in_dtype == POS_IN_BF16)
      pack_mc_kernel<bf, false, kFlag, kUC><<<grid, 256, 0, s>>>(
          dc, wgb, off_slot, off_slot2, static_cast<const bf*>(u), static_cast<const bf*>(v), M, N,
          Mp, R, K, gf, P);
    else
      pack_mc_kernel<float, false, kFlag, kUC><<<grid, 256, 0, s>>>(
          dc, wgb, off_slot, off_slot2, static_cast<const float*>(u),
          static_cast<const float*>(v), M, N, Mp, R, K, gf, P);
  }
}
}  // namespace

int symm_pack_mc(pos_ctx* c, int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                 const void* u, const void* v, void* gbuf, cudaStream_t s, bool* done,
                 void* gbuf2, uint32_t* flags, unsigned* fstate) {
  clear_stale_launch_error();
  *done = false;
  if (c->world < 2 || c->local) return POS_OK;
  static const bool mc_off = [] {   // POS_PACK_MC=0: pack locally + NCCL all-gather instead
    const char* e = getenv("POS_PACK_MC");
    return e && e[0] == '0';
  }();
  if (mc_off) return POS_OK;
  const int64_t R = row_elems(M, N), eb = dtype_bytes(dtype);
  const size_t slot_bytes = (size_t)(K * R * eb);
  ncclWindow_t wgb, wgb2, wfl;
  size_t off, off2 = 0, offf = 0;
  if (!symm_lookup(c, gbuf, slot_bytes * c->world, &wgb, &off)) return POS_OK;
  // flag mode needs the second buffer in the same window as the first (one window argument)
  const bool flag_mode = gbuf2 && flags && fstate &&
                         symm_lookup(c, gbuf2, slot_bytes * c->world, &wgb2, &off2) &&
                         symm_lookup(c, flags, sizeof(uint32_t) * c->world, &wfl, &offf);
  if (gbuf2 && !flag_mode) return POS_OK;   // inconsistent registration: caller uses NCCL
  const size_t off_slot = off + (size_t)c->rank * slot_bytes;
  const int vec = dtype == POS_DT_BF16 ? 8 : 4;
  // barrier mode: one LSA barrier index per CTA (<= kBarriers); flag mode: no barrier, more CTAs
  // keep more multicast stores in flight
  static const int pack_ctas = [] {
    const char* e = getenv("POS_PACK_CTAS");
    const int v = (e && *e) ? atoi(e) : 128;
    return v < 1 ? 1 : v;
  }();
  static const int pack_ctas_flag = [] {
    const char* e = getenv("POS_PACK_CTAS_FLAG");
    const int v = (e && *e) ? atoi(e) : 128;
    return v < 1 ? 1 : v;
  }();
  const int grid = grid_for(K * (R / vec), 256,
                            flag_mode ? pack_ctas_flag : std::min(pack_ctas, kBarriers));
  const int64_t Mp = m_pad(M);
  const ncclDevComm& dc = state(c)->dev;
  if (flag_mode) {
    // both buffers must be addressable through the first buffer's window: they are separate
    // allocations, so pass the second one's window offset relative to its own window instead
    GatherFlags gf{wfl, offf + sizeof(uint32_t) * (size_t)c->rank, fstate};
    if (wgb2 != wgb) return POS_OK;         // (separate windows: not supported, NCCL path)
    static const bool uc = [] {
      const char* e = getenv("POS_PACK_UC");
      return e && e[0] == '1';
    }();
    if (uc && c->world <= 8)
      launch_pack_mc<true, true>(grid, s, dc, wgb, off_slot, off2 + (size_t)c->rank * slot_bytes,
                                 in_dtype, dtype, u, v, M, N, Mp, R, K, gf, c->world);
    else
      launch_pack_mc<true>(grid, s, dc, wgb, off_slot, off2 + (size_t)c->rank * slot_bytes,
                           in_dtype, dtype, u, v, M, N, Mp, R, K, gf);
  } else {
    launch_pack_mc<false>(grid, s, dc, wgb, off_slot, off_slot, in_dtype, dtype, u, v, M, N, Mp,
                          R, K, GatherFlags{});
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "pack_mc_kernel launch");
  *done = true;
  return POS_OK;
}

int symm_wait_gathered(pos_ctx* c, const uint32_t* flags, const unsigned* fstate,
                       cudaStream_t s) {
  clear_stale_launch_error();
  wait_flags_kernel<<<1, 32, 0, s>>>(flags, fstate, c->world);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return ctx_cuda_fail(c, e, "wait_flags_kernel launch");
  return POS_OK;
}

}  // namespace pos

using namespace pos;

extern "C" {

int pos_mem_alloc(pos_ctx* c, int64_t bytes, void** out) {
  clear_error();
  POS_CHECK_ARG(c && out && bytes > 0, "bad arguments");
  int rc = symm_init(c);
  if (rc) return rc;
  void* p = nullptr;
  ncclResult_t r = ncclMemAlloc(&p, (size_t)bytes);
  if (r != ncclSuccess) return ctx_nccl_fail(c, r, "ncclMemAlloc");
  ncclWindow_t win;
  r = ncclCommWindowRegister(c->comm, p, (size_t)bytes, &win, NCCL_WIN_COLL_SYMMETRIC);
  if (r != ncclSuccess) {
    ncclMemFree(p);
    return ctx_nccl_fail(c, r, "ncclCommWindowRegister");
  }
  state(c)->windows.push_back({static_cast<char*>(p), (size_t)bytes, win});
  // NCCL's allocation/registration may leave a benign runtime error behind: consume it so it is
  // not misreported by the next kernel-launch check
  (void)cudaGetLastError();
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
  ncclWindow_t w;
  size_t off;
  return (c && symm_lookup(c, p, (size_t)bytes, &w, &off)) ? 1 : 0;
}

}  // extern "C"
