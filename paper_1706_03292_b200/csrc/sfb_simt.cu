// A4 fallback: SFB reconstruct-and-apply on the CUDA cores, for a W the TMA path cannot address
// (N % 4 != 0, ldw % 4 != 0 or W not 16-byte aligned), any dtype.
//   W[m][n] = (accumulate ? W[m][n] : 0) + alpha * sum_{j<KP} U[j][m] * V[j][n]
// over KP gathered ROWS (for POS_DT_F32 the 3xTF32 rows: the same three-term sum the tensor-core
// path takes, reading S16). Shared-memory tiled FFMA GEMM, fp32 accumulation in a fixed k order.
// (Round 1-2 ran POS_DT_F32 here for every shape: 340 us for VGG fc6 at K*P = 32, 0.37 of HBM.)
// Tile 128 x 128, BK 16, 256 threads, 8 x 8 outputs per thread.
#include <cuda_bf16.h>

#include "common.h"

namespace pos {
namespace {

constexpr int TM = 128, TN = 128, TK = 16, THREADS = 256;

__device__ __forceinline__ float ld_g(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float ld_g(const float* p) { return *p; }

template <typename T>
__global__ void __launch_bounds__(THREADS)
sfb_simt_kernel(const T* __restrict__ U, const T* __restrict__ V, int64_t R, int64_t M, int64_t N,
                int64_t KP, int accumulate, float* __restrict__ W, int64_t ldw, float alpha) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.y * TM, n0 = (int64_t)blockIdx.x * TN;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  for (int64_t k0 = 0; k0 < KP; k0 += TK) {
    // cooperative load: TK x 128 for A (rows of U) and B (rows of V); 8 elements per thread each
#pragma unroll
    for (int r = 0; r < (TK * TM) / THREADS; ++r) {
      const int e = tid + r * THREADS;
      const int kk = e / TM, c = e % TM;
      const int64_t k = k0 + kk;
      const int64_t m = m0 + c, n = n0 + c;
      As[kk][c] = (k < KP && m < M) ? ld_g(U + k * R + m) : 0.0f;
      Bs[kk][c] = (k < KP && n < N) ? ld_g(V + k * R + n) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t m = m0 + ty + 16 * i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t n = n0 + tx + 16 * j;
      if (n < N) {
        float* p = W + m * ldw + n;
        const float base = accumulate ? *p : 0.0f;
        *p = fmaf(alpha, acc[i][j], base);
      }
    }
  }
}

}  // namespace

cudaError_t launch_sfb_simt(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                            int32_t accumulate, float* W, int64_t ldw, float alpha,
                            cudaStream_t s) {
  clear_stale_launch_error();
  const int64_t R = row_elems(M, N), Mp = m_pad(M);
  const int64_t gy = (M + TM - 1) / TM, gx = (N + TN - 1) / TN;
  if (gy > 65535) return cudaErrorInvalidValue;
  dim3 grid((unsigned)gx, (unsigned)gy);
  if (dtype == POS_DT_BF16) {
    auto* g = static_cast<const __nv_bfloat16*>(G);
    sfb_simt_kernel<<<grid, THREADS, 0, s>>>(g, g + Mp, R, M, N, KP, accumulate, W, ldw, alpha);
  } else {
    auto* g = static_cast<const float*>(G);
    sfb_simt_kernel<<<grid, THREADS, 0, s>>>(g, g + Mp, R, M, N, KP, accumulate, W, ldw, alpha);
  }
  return cudaGetLastError();
}


cudaError_t preload_simt_kernels() {
  cudaFuncAttributes fa;
  if (cudaError_t e = cudaFuncGetAttributes(&fa, sfb_simt_kernel<__nv_bfloat16>); e != cudaSuccess) return e;
  return cudaFuncGetAttributes(&fa, sfb_simt_kernel<float>);
}

}  // namespace pos
