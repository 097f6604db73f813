// HBM-bound kernels of the hot path:
//   A2  factor pack      u, v (autograd layout) -> gathered row [u | 0 pad | v | 1, 0 pad] in dtype
//   A4b bias column sum  b (+)= alpha * sum_j U[j][m], fixed order (deterministic)
//   A7  PS shard apply   W += alpha * g, 16-byte vectors, grid-stride
//   sim PS reduce-apply  W += alpha * sum_p g_p (the simulated-P stand-in for RS + A7 + AG)
// Roofline: all of these are bound by HBM bandwidth; they are coalesced and 16-byte vectorised
// on the side that dominates the traffic.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.h"

namespace pos {
namespace {

__device__ __forceinline__ float ld_in(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_in(const float* p) { return *p; }
// ---------------------------------------------------------------------------------------------
// A2: one thread writes one 16-byte output vector. grid.y = sample row k (K <= 65535 per launch
// chunk). The input rows are read with plain (unaligned-safe) loads; consecutive threads read
// consecutive elements, so the reads coalesce.
// ---------------------------------------------------------------------------------------------
template <typename Tin, bool kBF16>
__global__ void pack_kernel(const Tin* __restrict__ u, const Tin* __restrict__ v,
                            void* __restrict__ out, int64_t M, int64_t N, int64_t Mp, int64_t R,
                            int64_t r0, int64_t K, int split) {
  constexpr int VEC = kBF16 ? 8 : 4;
  const int64_t r = r0 + blockIdx.y;                                  // gathered row
  const int64_t k = split ? r % K : r;                                // its factor pair
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // VEC-element chunk in row
  const int64_t col = c * VEC;
  if (col >= R) return;
  const Tin* src;
  int64_t idx, lim;
  if (col < Mp) { src = u + k * M; idx = col; lim = M; }
  else          { src = v + k * N; idx = col - Mp; lim = N; }
  // v's first pad column (index N) holds 1.0: the reconstruction's extra output column is then
  // sum_j u_j, the bias gradient (A4b fused into A4); every other pad element is 0
  const int64_t onec = col < Mp ? -1 : N;
  const int64_t eb = kBF16 ? 2 : 4;
  uint4 q = pack_chunk<Tin, kBF16>(src, idx, lim, onec);
  if constexpr (!kBF16)
    if (split) q = tf32_split4(q, split_part(r / K, col >= Mp));
  *reinterpret_cast<uint4*>(static_cast<char*>(out) + (r * R + col) * eb) = q;
}

// ---------------------------------------------------------------------------------------------
// A4b: block = 32 columns x 8 warps. Warp w sums the contiguous row range [w*chunk, (w+1)*chunk)
// for its lane's column; the 8 partials are then added in warp order. Fixed order => bitwise
// reproducible; every rank computes the same value from the same gathered U. Each row is weighted
// by its ones-column entry (column onec = M_pad + N): 1 everywhere except the (hi u, lo v) block
// of a 3xTF32 slot, where it is 0 — the same sum the tensor-core path takes from column N.
// ---------------------------------------------------------------------------------------------
template <typename T>
__global__ void bias_colsum_kernel(const T* __restrict__ G, int64_t M, int64_t R, int64_t KP,
                                   int64_t onec, int accumulate, float* __restrict__ b,
                                   float alpha) {
  __shared__ float part[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t m = (int64_t)blockIdx.x * 32 + lane;
  const int64_t chunk = (KP + 7) / 8;
  const int64_t j0 = w * chunk, j1 = min(KP, j0 + chunk);
  float s = 0.0f;
  if (m < M)
    for (int64_t j = j0; j < j1; ++j) s = fmaf(ld_in(G + j * R + m), ld_in(G + j * R + onec), s);
  part[w][lane] = s;
  __syncthreads();
  if (w == 0 && m < M) {
    float t = part[0][lane];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += part[i][lane];
    const float base = accumulate ? b[m] : 0.0f;
    b[m] = fmaf(alpha, t, base);
  }
}

// ---------------------------------------------------------------------------------------------
// A7: W += alpha * g. Each thread moves UNROLL float4 per iteration with all loads issued first.
// ---------------------------------------------------------------------------------------------
constexpr int kApplyUnroll = 4;

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__global__ void ps_apply_vec_kernel(const float4* __restrict__ g, float4* __restrict__ W,
                                    int64_t n4, float alpha, KTrace tr, KTrace tg) {
  ktrace_begin(tr);
  ktrace_begin(tg);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (kApplyUnroll - 1) * stride < n4; i += kApplyUnroll * stride) {
    float4 gv[kApplyUnroll], wv[kApplyUnroll];
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) {
      gv[u] = ld_stream(g + i + u * stride);
      wv[u] = W[i + u * stride];
    }
#pragma unroll
    for (int u = 0; u < kApplyUnroll; ++u) {
      wv[u].x = fmaf(alpha, gv[u].x, wv[u].x);
      wv[u].y = fmaf(alpha, gv[u].y, wv[u].y);
      wv[u].z = fmaf(alpha, gv[u].z, wv[u].z);
      wv[u].w = fmaf(alpha, gv[u].w, wv[u].w);
      W[i + u * stride] = wv[u];
    }
  }
  for (; i < n4; i += stride) {
    float4 gv = ld_stream(g + i), wv = W[i];
    wv.x = fmaf(alpha, gv.x, wv.x);
    wv.y = fmaf(alpha, gv.y, wv.y);
    wv.z = fmaf(alpha, gv.z, wv.z);
    wv.w = fmaf(alpha, gv.w, wv.w);
    W[i] = wv;
  }
  if (tr.rec || tg.rec) {
    __syncthreads();
    ktrace_end(tr);
    ktrace_end(tg);
  }
}

__global__ void ps_apply_scalar_kernel(const float* __restrict__ g, float* __restrict__ W,
                                       int64_t n, float alpha) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    W[i] = fmaf(alpha, g[i], W[i]);
}

struct GradPtrs {
  const float* p[kMaxSimP];
};

// Simulated reduce-scatter + apply + all-gather on one GPU: the P gradients are summed in worker
// order (what a reduction over P ranks computes), then applied.
__global__ void sim_ps_reduce_apply_kernel(GradPtrs gp, int P, float* __restrict__ W, int64_t n,
                                           float alpha) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float s = gp.p[0][i];
    for (int p = 1; p < P; ++p) s += gp.p[p][i];
    W[i] = fmaf(alpha, s, W[i]);
  }
}

int grid_for(int64_t work_items, int threads) {
  int64_t blocks = (work_items + threads - 1) / threads;
  static const int64_t mult = [] {   // CTAs per SM cap of the streaming kernels
    const char* e = getenv("POS_STREAM_CTAS_PER_SM");
    const int v = (e && *e) ? atoi(e) : 8;
    return (int64_t)(v < 1 ? 1 : v);
  }();
  const int64_t cap = (int64_t)num_sms() * mult;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace

cudaError_t launch_pack_factors(int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                                const void* u, const void* v, void* slot, cudaStream_t s) {
  clear_stale_launch_error();
  const int64_t Mp = m_pad(M), R = row_elems(M, N);
  const int threads = 128;
  const int vec = dtype == POS_DT_BF16 ? 8 : 4;
  const int64_t chunks = R / vec;
  const int64_t rows = K * rows_per_sample(dtype);
  const int split = rows_per_sample(dtype) == 3;
  for (int64_t r0 = 0; r0 < rows; r0 += 65535) {
    const unsigned nr = (unsigned)std::min<int64_t>(65535, rows - r0);
    dim3 grid((unsigned)((chunks + threads - 1) / threads), nr);
    using bf = __nv_bfloat16;
    const bool in_bf = in_dtype == POS_IN_BF16;
    if (dtype == POS_DT_BF16) {
      if (in_bf) pack_kernel<bf, true><<<grid, threads, 0, s>>>(static_cast<const bf*>(u), static_cast<const bf*>(v), slot, M, N, Mp, R, r0, K, 0);
      else       pack_kernel<float, true><<<grid, threads, 0, s>>>(static_cast<const float*>(u), static_cast<const float*>(v), slot, M, N, Mp, R, r0, K, 0);
    } else {
      if (in_bf) pack_kernel<bf, false><<<grid, threads, 0, s>>>(static_cast<const bf*>(u), static_cast<const bf*>(v), slot, M, N, Mp, R, r0, K, split);
      else       pack_kernel<float, false><<<grid, threads, 0, s>>>(static_cast<const float*>(u), static_cast<const float*>(v), slot, M, N, Mp, R, r0, K, split);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_bias_colsum(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                               int32_t accumulate, float* b, float alpha, cudaStream_t s) {
  clear_stale_launch_error();
  const int64_t R = row_elems(M, N), onec = m_pad(M) + N;
  const unsigned blocks = (unsigned)((M + 31) / 32);
  if (dtype == POS_DT_BF16)
    bias_colsum_kernel<<<blocks, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(G), M, R, KP, onec,
                                              accumulate, b, alpha);
  else
    bias_colsum_kernel<<<blocks, 256, 0, s>>>(static_cast<const float*>(G), M, R, KP, onec,
                                              accumulate, b, alpha);
  return cudaGetLastError();
}

int ps_apply_grid(int64_t count) {
  const int64_t n4 = count / 4;
  return n4 > 0 ? grid_for((n4 + kApplyUnroll - 1) / kApplyUnroll, 256) : 0;
}

cudaError_t launch_ps_apply(const float* g, float* W, int64_t count, float alpha, cudaStream_t s,
                            KTrace tr, KTrace tg) {
  clear_stale_launch_error();
  const int threads = 256;
  if (aligned16(g) && aligned16(W)) {
    const int64_t n4 = count / 4;
    const int grid = ps_apply_grid(count);
    if (tr.rec && tr.expected == 0) tr.expected = (unsigned)grid;
    if (n4 > 0)
      ps_apply_vec_kernel<<<grid, threads, 0, s>>>(reinterpret_cast<const float4*>(g),
                                                   reinterpret_cast<float4*>(W), n4, alpha, tr, tg);
    const int64_t rem = count - n4 * 4;
    if (rem > 0)
      ps_apply_scalar_kernel<<<1, 32, 0, s>>>(g + n4 * 4, W + n4 * 4, rem, alpha);
  } else {
    ps_apply_scalar_kernel<<<grid_for(count, threads), threads, 0, s>>>(g, W, count, alpha);
  }
  return cudaGetLastError();
}

cudaError_t launch_sim_ps_reduce_apply(const float* const* grads, int P, float* W, int64_t n,
                                       float alpha, cudaStream_t s) {
  clear_stale_launch_error();
  GradPtrs gp{};
  for (int p = 0; p < P; ++p) gp.p[p] = grads[p];
  const int threads = 256;
  sim_ps_reduce_apply_kernel<<<grid_for(n, threads), threads, 0, s>>>(gp, P, W, n, alpha);
  return cudaGetLastError();
}

__global__ void ktrace_init_kernel(unsigned long long* rec) {
  if (threadIdx.x < kTraceWords) rec[threadIdx.x] = threadIdx.x == 0 ? ~0ull : 0ull;
}

cudaError_t ktrace_alloc(unsigned long long** rec) {
  cudaError_t e = cudaMalloc(rec, kTraceWords * sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  return ktrace_reset(*rec);
}

cudaError_t ktrace_reset(unsigned long long* rec) {
  clear_stale_launch_error();
  ktrace_init_kernel<<<1, 32>>>(rec);
  cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? e : cudaDeviceSynchronize();
}

cudaError_t preload_mem_kernels() {
  using bf = __nv_bfloat16;
  cudaFuncAttributes fa;
  const void* fns[] = {
      reinterpret_cast<const void*>(pack_kernel<bf, true>), reinterpret_cast<const void*>(pack_kernel<float, true>),
      reinterpret_cast<const void*>(pack_kernel<bf, false>), reinterpret_cast<const void*>(pack_kernel<float, false>),
      reinterpret_cast<const void*>(bias_colsum_kernel<bf>), reinterpret_cast<const void*>(bias_colsum_kernel<float>),
      reinterpret_cast<const void*>(ps_apply_vec_kernel), reinterpret_cast<const void*>(ps_apply_scalar_kernel),
      reinterpret_cast<const void*>(sim_ps_reduce_apply_kernel), reinterpret_cast<const void*>(ktrace_init_kernel)};
  for (const void* f : fns)
    if (cudaError_t e = cudaFuncGetAttributes(&fa, f); e != cudaSuccess) return e;
  return cudaSuccess;
}

}  // namespace pos
