// A4 — SFB reconstruct-and-apply on the 5th-generation tensor cores (sm_100a).
//
//   W[m][n] = (accumulate ? W[m][n] : 0) + alpha * sum_{j < KP} U[j][m] * V[j][n]
//
// PAPER:111 §2.1: the FC gradient of one sample is u v^T, and SFB "reconstruct[s] the gradient
// matrices using u, v locally"; Eq. 2 sums the P workers' batches. With the K*P
// gathered factor rows stacked as U (KP x M) and V (KP x N) that is the dense contraction
// U^T V with inner dimension KP, fused here with the SGD apply of PAPER:107 ("apply (+)").
//
// Design:
//  * persistent, warp-specialised CTA, one per SM; 128 x 256 output tile; tiles handed out by a
//    dynamic atomic tile scheduler (or static round-robin); no split-K, no atomics on data: a
//    tile's arithmetic never depends on which CTA computes it -> bitwise-identical replicas;
//  * operands U, V streamed by TMA (128-byte swizzle, MN-major: m / n is the contiguous
//    direction of the gathered rows; 128-byte aligned rows) into a 3-stage smem ring, consumed
//    by tcgen05.mma issued by one thread, accumulating in TMEM (fp32). Two 256-column TMEM
//    accumulators: the epilogue of tile i overlaps the MMAs of tile i+1;
//  * the W tile (the HBM-dominant traffic: 8 bytes per element) is streamed in 128 x 32 fp32
//    sub-tiles by a second TMA producer warp into a 5-slot ring, updated in shared memory by the
//    4 epilogue warps (tcgen05.ld 32x32b -> fma -> st.shared) and written back by TMA store;
//  * the bias gradient comes out of the same GEMM: the packed v rows carry a 1.0 in column N,
//    so accumulator column N is sum_j u_j (A4b fused; read with one tcgen05.ld 32x32b.x1).
//
// Warp roles (256 threads): w0 operand TMA producer, w1 MMA issuer + TMEM owner, w2 W TMA
// producer, w3 idle, w4..w7 epilogue (warp w%4 owns TMEM lanes 32*(w%4) .. +31 = tile rows).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.h"

namespace pos {
namespace {

constexpr int BM = 128;             // tile rows (m) = UMMA M = TMEM lanes
#ifndef POS_SFB_BN
#define POS_SFB_BN 256
#endif
constexpr int BN = POS_SFB_BN;      // tile cols (n) = UMMA N = TMEM columns per accumulator
#ifndef POS_SFB_STAGES
#define POS_SFB_STAGES 3
#endif
#ifndef POS_SFB_WSLOTS
#define POS_SFB_WSLOTS 5
#endif
// The kernel is bound by the W read-modify-write (8 B per element): shared memory goes to W
// prefetch depth (WSLOTS x 16 KB in flight per SM) rather than to operand stages (K*P is small).
constexpr int STAGES = POS_SFB_STAGES;   // operand ring depth
constexpr int WSLOTS = POS_SFB_WSLOTS;   // W sub-tile ring depth
constexpr int WSUB = 32;            // W sub-tile columns (32 fp32 = one 128-byte swizzle row)
constexpr int NSUB = BN / WSUB;     // sub-tiles per tile
constexpr int SWZ = 128;            // swizzle span in bytes (one operand "row" chunk)
#ifndef POS_SFB_KBYTES
#define POS_SFB_KBYTES 128
#endif
constexpr int KBYTES = POS_SFB_KBYTES;   // bytes of K per operand row per stage (BK = KBYTES / elt)
constexpr int A_BYTES = KBYTES * BM;     // per stage: BK rows x BM elements (any dtype)
constexpr int B_BYTES = KBYTES * BN;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int W_BYTES = BM * WSUB * 4;
constexpr int SMEM_DATA = STAGES * STAGE_BYTES + WSLOTS * W_BYTES;
constexpr int TR = 4;               // tile-index ring depth (dynamic tile scheduler)
constexpr int SMEM_BARS = 8 * (2 * STAGES + 2 * WSLOTS + 4 + 2 * TR) + 16 + 4 * TR;
constexpr int SMEM_TOTAL = SMEM_DATA + SMEM_BARS + 1024;   // + alignment slack
constexpr int THREADS = 256;
constexpr int TMEM_COLS = 2 * BN;

static_assert(SMEM_TOTAL <= 232448, "shared memory budget");

// ------------------------------------------------------------------------------------ PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint32_t bar, uint32_t dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int32_t c0,
                                             int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];"
               ::"l"(map), "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
// L2 cache-policy variants: W is streamed exactly once (evict first, so it does not displace the
// operands U, V that every CTA re-reads; its dirty lines also leave L2 sooner).
#ifndef POS_SFB_L2HINT
#define POS_SFB_L2HINT 0
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_hint(const CUtensorMap* map, uint32_t bar,
                                                 uint32_t dst, int32_t c0, int32_t c1,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, uint32_t src,
                                                  int32_t c0, int32_t c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group.L2::cache_hint"
      " [%0, {%1, %2}], [%3], %4;" ::"l"(map), "r"(c0), "r"(c1), "r"(src), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, one elected thread issues for the whole CTA.
template <bool kTF32>
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                     uint32_t idesc, uint32_t accumulate) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
// mbarrier arrives when all previously issued tcgen05 ops of this thread have completed
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor, version 1 (sm_100). For MN-major operands the leading byte
// offset (LBO) is the distance between 128-byte chunks along M/N and the stride byte offset (SBO)
// the distance between swizzle-atom row groups along K.
//   16-bit operands: SWIZZLE_128B (layout 2) — 16-byte granules, 8-row atoms (SBO = 1024 B);
//   32-bit (tf32) MN-major operands: SWIZZLE_128B_BASE32B (layout 1) — 32-byte granules, 4-row
//   atoms (SBO = 512 B); the only MN-major smem layout the tensor core accepts for tf32.
template <bool kTF32>
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo) {
  constexpr uint32_t sbo = kTF32 ? 4 * 128 : 8 * 128;
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;                   // descriptor version (sm_100)
  d |= (uint64_t)(kTF32 ? 1 : 2) << 61;     // layout type
  return d;
}

// Instruction descriptor: fp32 accumulate, A/B format (BF16 = 1, TF32 = 2), both MN-major,
// N = BN, M = BM.
template <bool kTF32>
__host__ __device__ constexpr uint32_t instr_desc() {
  return (1u << 4) | ((kTF32 ? 2u : 1u) << 7) | ((kTF32 ? 2u : 1u) << 10) | (1u << 15) |
         (1u << 16) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// number of W sub-tiles of the tile starting at column n0 that intersect [0, N)
__device__ __forceinline__ int nsub_of(int64_t N, int n0) {
  const int64_t s = (N - n0 + WSUB - 1) / WSUB;
  return s < NSUB ? (int)s : NSUB;
}

struct TileInfo {
  int64_t M, N, KP;
  int nb_n;        // tiles along n
  int num_tiles;
  int nkb;         // k blocks
  // Dynamic tile scheduler: [0] = next tile, [1] = CTAs finished. nullptr = static round-robin.
  // Self-resetting: the last CTA to finish zeroes both, so the counter is reusable by the next
  // launch on the same stream (and by every CUDA-graph replay).
  unsigned int* counter;
  float* bias;     // fused A4b: b (+)= alpha * accumulator column N; nullptr = no bias
};

template <bool kTF32>
__global__ void __launch_bounds__(THREADS, 1)
sfb_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmW, TileInfo ti, float alpha, int accumulate) {
  constexpr int EB = kTF32 ? 4 : 2;          // element bytes
  constexpr int BK = KBYTES / EB;            // k rows per stage (64 bf16 / 32 tf32 at 128 B)
  constexpr int CHUNK = SWZ / EB;            // elements per 128-byte chunk along m / n
  constexpr int UK = 32 / EB;                // UMMA K (16 bf16 / 8 tf32)
  constexpr int BOX_BYTES = BK * SWZ;        // one TMA box: BK rows x 128 B
  constexpr uint32_t IDESC = instr_desc<kTF32>();

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sW0 = sbase + STAGES * STAGE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SMEM_DATA);
  const uint32_t b_full = smem_u32(bars), b_empty = b_full + 8 * STAGES;
  const uint32_t b_wfull = b_empty + 8 * STAGES, b_wempty = b_wfull + 8 * WSLOTS;
  const uint32_t b_tfull = b_wempty + 8 * WSLOTS, b_tempty = b_tfull + 16;
  const uint32_t b_rfull = b_tempty + 16, b_rempty = b_rfull + 8 * TR;   // tile-index ring
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 2 * WSLOTS + 4 + 2 * TR);
  volatile int* tile_ring = reinterpret_cast<volatile int*>(tmem_slot + 4);
  const bool dyn = ti.counter != nullptr;
  // The tile sequence every role walks: static round-robin, or the fetcher's atomic sequence
  // broadcast through the ring (it -> tile, -1 = done). All roles see the same sequence.
  auto tile_of = [&](int it, uint32_t& rphase) -> int {
    if (!dyn) {
      const int t = blockIdx.x + it * gridDim.x;
      return t < ti.num_tiles ? t : -1;
    }
    const int slot = it % TR;
    mbar_wait(b_rfull + 8 * slot, rphase);
    const int t = tile_ring[slot];
    mbar_arrive(b_rempty + 8 * slot);
    if (slot == TR - 1) rphase ^= 1;
    return t;
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) { mbar_init(b_full + 8 * i, 1); mbar_init(b_empty + 8 * i, 1); }
    for (int i = 0; i < WSLOTS; ++i) { mbar_init(b_wfull + 8 * i, 1); mbar_init(b_wempty + 8 * i, 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(b_tfull + 8 * i, 1); mbar_init(b_tempty + 8 * i, 128); }
    // ring consumers: MMA issuer + W producer + 128 epilogue threads
    for (int i = 0; i < TR; ++i) { mbar_init(b_rfull + 8 * i, 1); mbar_init(b_rempty + 8 * i, 130); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== operand TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, rphase = 0;
      for (int it = 0;; ++it) {
        int t;
        if (!dyn) {
          t = blockIdx.x + it * gridDim.x;
          if (t >= ti.num_tiles) break;
        } else {   // fetch the next tile and publish it to the other roles
          const int slot = it % TR;
          mbar_wait(b_rempty + 8 * slot, rphase ^ 1);
          t = (int)atomicAdd(ti.counter, 1u);
          if (t >= ti.num_tiles) t = -1;
          tile_ring[slot] = t;
          mbar_arrive(b_rfull + 8 * slot);
          if (slot == TR - 1) rphase ^= 1;
          if (t < 0) {
            __threadfence();
            if (atomicAdd(ti.counter + 1, 1u) == gridDim.x - 1) {   // last CTA out resets
              ti.counter[0] = 0;
              ti.counter[1] = 0;
              __threadfence();
            }
            break;
          }
        }
        const int m0 = (t / ti.nb_n) * BM, n0 = (t % ti.nb_n) * BN;
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(b_empty + 8 * stage, phase ^ 1);
          const uint32_t full = b_full + 8 * stage;
          mbar_expect_tx(full, STAGE_BYTES);
          const uint32_t sA = sbase + stage * STAGE_BYTES, sB = sA + A_BYTES;
          const int k0 = kb * BK;
#pragma unroll
          for (int c = 0; c < BM / CHUNK; ++c) tma_load_2d(&tmA, full, sA + c * BOX_BYTES, m0 + c * CHUNK, k0);
#pragma unroll
          for (int c = 0; c < BN / CHUNK; ++c) tma_load_2d(&tmB, full, sB + c * BOX_BYTES, n0 + c * CHUNK, k0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0, rphase = 0;
      for (int it = 0;; ++it) {
        const int t = tile_of(it, rphase);
        if (t < 0) break;
        mbar_wait(b_tempty + 8 * acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(b_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t sA = sbase + stage * STAGE_BYTES, sB = sA + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = smem_desc<kTF32>(sA + kk * UK * SWZ, BOX_BYTES);
            const uint64_t bd = smem_desc<kTF32>(sB + kk * UK * SWZ, BOX_BYTES);
            umma<kTF32>(d_tmem, ad, bd, IDESC, (kb | kk) != 0);
          }
          umma_commit(b_empty + 8 * stage);   // frees the smem stage when these MMAs finish
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(b_tfull + 8 * acc);        // accumulator ready for the epilogue
        if (++acc == 2) { acc = 0; aphase ^= 1; }
      }
    }
  } else if (warp == 2) {
    // ===================== W sub-tile TMA producer =====================
    if (lane == 0) {
      int ws = 0;
      uint32_t wphase = 0, rphase = 0;
      for (int it = 0;; ++it) {
        const int t = tile_of(it, rphase);
        if (t < 0) break;
        const int m0 = (t / ti.nb_n) * BM, n0 = (t % ti.nb_n) * BN;
        const int nsub = nsub_of(ti.N, n0);
        for (int j = 0; j < nsub; ++j) {
          mbar_wait(b_wempty + 8 * ws, wphase ^ 1);
          const uint32_t wf = b_wfull + 8 * ws;
          if (accumulate) {
            mbar_expect_tx(wf, W_BYTES);
            if (POS_SFB_L2HINT)
              tma_load_2d_hint(&tmW, wf, sW0 + ws * W_BYTES, n0 + j * WSUB, m0, policy_evict_first());
            else
              tma_load_2d(&tmW, wf, sW0 + ws * W_BYTES, n0 + j * WSUB, m0);
          } else {
            mbar_arrive(wf);
          }
          if (++ws == WSLOTS) { ws = 0; wphase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> regs, W += alpha * acc in smem, TMA store ========
    const int et = threadIdx.x - 128;         // tile row owned by this thread
    const int q = warp & 3;                   // TMEM lane quadrant of this warp
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    int acc = 0;
    uint32_t aphase = 0;
    int ws = 0;
    uint32_t wphase = 0;
    int pending = -1;                         // slot whose TMA store has not been retired yet
    uint32_t rphase = 0;
    for (int it = 0;; ++it) {
      const int t = tile_of(it, rphase);
      if (t < 0) break;
      const int m0 = (t / ti.nb_n) * BM, n0 = (t % ti.nb_n) * BN;
      const int nsub = nsub_of(ti.N, n0);
      mbar_wait(b_tfull + 8 * acc, aphase);
      tc_fence_after();
      // A4b fused: the gathered v rows carry a 1.0 in column N, so accumulator column N of the
      // tile holding it is sum_j U[j][m] — the bias gradient of row m
      if (ti.bias && (int64_t)n0 <= ti.N && ti.N < (int64_t)n0 + BN) {
        uint32_t bv;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                     : "=r"(bv)
                     : "r"(tmem_base + lane_addr + acc * BN + (uint32_t)(ti.N - n0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int64_t m = (int64_t)m0 + et;
        if (m < ti.M) {
          const float base = accumulate ? ti.bias[m] : 0.0f;
          ti.bias[m] = fmaf(alpha, __uint_as_float(bv), base);
        }
      }
      if (nsub == 0) {                        // bias-only tile: nothing else reads TMEM
        tc_fence_before();
        mbar_arrive(b_tempty + 8 * acc);
      }
      for (int j = 0; j < nsub; ++j) {
        uint32_t r[32];
        tmem_ld32(tmem_base + lane_addr + acc * BN + j * WSUB, r);
        if (j == nsub - 1) {                  // accumulator fully drained by this thread
          tc_fence_before();
          mbar_arrive(b_tempty + 8 * acc);
        }
        mbar_wait(b_wfull + 8 * ws, wphase);
        const uint32_t row = sW0 + ws * W_BYTES + et * SWZ;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t a = row + ((uint32_t)(c ^ (et & 7)) << 4);   // 128-byte swizzle
          float4 w;
          if (accumulate) {
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(w.x), "=f"(w.y), "=f"(w.z), "=f"(w.w) : "r"(a));
          } else {
            w = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          w.x = fmaf(alpha, __uint_as_float(r[4 * c + 0]), w.x);
          w.y = fmaf(alpha, __uint_as_float(r[4 * c + 1]), w.y);
          w.z = fmaf(alpha, __uint_as_float(r[4 * c + 2]), w.z);
          w.w = fmaf(alpha, __uint_as_float(r[4 * c + 3]), w.w);
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(w.x), "f"(w.y),
                       "f"(w.z), "f"(w.w)
                       : "memory");
        }
        fence_proxy_async_smem();             // generic-proxy smem writes -> visible to TMA
        named_bar_sync(1, 128);
        if (et == 0) {
          if (POS_SFB_L2HINT)
            tma_store_2d_hint(&tmW, sW0 + ws * W_BYTES, n0 + j * WSUB, m0, policy_evict_first());
          else
            tma_store_2d(&tmW, sW0 + ws * W_BYTES, n0 + j * WSUB, m0);
          bulk_commit();
          if (pending >= 0) {
            bulk_wait_read<1>();              // the previous store has finished reading smem
            mbar_arrive(b_wempty + 8 * pending);
          }
          pending = ws;
        }
        if (++ws == WSLOTS) { ws = 0; wphase ^= 1; }
      }
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (et == 0) bulk_wait_all();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "n"(TMEM_COLS)
                 : "memory");
  }
}

// ------------------------------------------------------------------------ host side ----------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner,
               uint64_t outer, uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool kTF32>
bool make_plan_impl(SfbTcPlan* pl, int64_t M, int64_t N, int64_t KP, const void* G, float* W,
                    int64_t ldw, int max_ctas, float* bias) {
  // with a bias the V operand includes the ones column N (the GEMM's extra output column)
  const int64_t NB = N + (bias ? 1 : 0);
  constexpr int EB = kTF32 ? 4 : 2;
  constexpr int BK = KBYTES / EB, CHUNK = SWZ / EB;
  const int64_t R = row_elems(M, N), Mp = m_pad(M);
  const CUtensorMapDataType dt =
      kTF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  // operand smem layout must match the UMMA descriptor (smem_desc<kTF32>)
  const CUtensorMapSwizzle oswz =
      kTF32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  const uint8_t* g = static_cast<const uint8_t*>(G);
  if (!encode_2d(&pl->tmA, dt, g, (uint64_t)M, (uint64_t)KP, (uint64_t)(R * EB), CHUNK, BK,
                 oswz) ||
      !encode_2d(&pl->tmB, dt, g + Mp * EB, (uint64_t)NB, (uint64_t)KP, (uint64_t)(R * EB),
                 CHUNK, BK, oswz) ||
      !encode_2d(&pl->tmW, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, W, (uint64_t)N, (uint64_t)M,
                 (uint64_t)(ldw * 4), WSUB, BM))
    return false;
  pl->M = M; pl->N = N; pl->KP = KP;
  pl->nb_n = (int)((NB + BN - 1) / BN);
  pl->bias = bias;
  const int64_t tiles = (int64_t)pl->nb_n * ((M + BM - 1) / BM);
  if (tiles > INT32_MAX) return false;
  pl->num_tiles = (int)tiles;
  pl->nkb = (int)((KP + BK - 1) / BK);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (grid > pl->num_tiles) grid = pl->num_tiles;
  pl->grid = grid;
  pl->tf32 = kTF32;
  return true;
}

template <bool kTF32>
cudaError_t launch_plan_impl(const SfbTcPlan& pl, float alpha, int accumulate, cudaStream_t s) {
  clear_stale_launch_error();
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(sfb_tc_kernel<kTF32>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  TileInfo ti;
  ti.M = pl.M; ti.N = pl.N; ti.KP = pl.KP;
  ti.nb_n = pl.nb_n; ti.num_tiles = pl.num_tiles; ti.nkb = pl.nkb;
  ti.counter = pl.counter;
  ti.bias = pl.bias;
  sfb_tc_kernel<kTF32><<<pl.grid, THREADS, SMEM_TOTAL, s>>>(pl.tmA, pl.tmB, pl.tmW, ti, alpha,
                                                              accumulate);
  return cudaGetLastError();
}

}  // namespace

bool sfb_tc_supported(int64_t N, int64_t ldw, const float* W, const void* G) {
  // TMA stores move whole 16-byte chunks: the last W row chunk must not straddle column N (else
  // the element(s) after N in a strided W would be overwritten) -> N % 4 == 0 as well as ldw.
  return (N % 4) == 0 && (ldw % 4) == 0 && aligned16(W) && aligned16(G) && N >= 1 &&
         get_encode() != nullptr;
}

bool sfb_tc_make_plan(SfbTcPlan* pl, int64_t M, int64_t N, int64_t KP, int32_t dtype,
                      const void* G, float* W, int64_t ldw, int max_ctas, float* bias) {
  if (dtype == POS_DT_F32 || !sfb_tc_supported(N, ldw, W, G)) return false;
  if (dtype == POS_DT_TF32) return make_plan_impl<true>(pl, M, N, KP, G, W, ldw, max_ctas, bias);
  return make_plan_impl<false>(pl, M, N, KP, G, W, ldw, max_ctas, bias);
}

cudaError_t sfb_tc_launch(const SfbTcPlan& pl, float alpha, int accumulate, cudaStream_t s) {
  return pl.tf32 ? launch_plan_impl<true>(pl, alpha, accumulate, s)
                 : launch_plan_impl<false>(pl, alpha, accumulate, s);
}

cudaError_t launch_sfb_tc(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                          int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                          int max_ctas, cudaStream_t s) {
  SfbTcPlan pl;
  if (!sfb_tc_make_plan(&pl, M, N, KP, dtype, G, W, ldw, max_ctas, b)) return cudaErrorInvalidValue;
  return sfb_tc_launch(pl, alpha, accumulate, s);
}

}  // namespace pos
