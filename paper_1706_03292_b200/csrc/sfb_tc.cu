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
//  * K*P >= 1024: CTA-pair variant (cluster of 2, tcgen05.mma.cta_group::2, M = 256): each CTA
//    stages its 128 rows of U and half of the tile's V columns, the even CTA issues the MMAs
//    for both; 1/3 less operand traffic and smaller stages (5 x 32 KB in flight + 4 W slots)
//    where the operand stream, not W, is the bound. At K*P = 1024 the kernel is bound by the
//    bytes each SM can keep in flight from L2 (operands 16 B + W 4 B per output element; the
//    diagnostic builds POS_SFB_EXP show MMA+operands alone at 0.95 of the tensor peak and the W
//    path alone at 0.92 of HBM — DESIGN.md §11). Measured and removed (round 2, commits 6664201,
//    7a655b0, 5d59ca3): 4-CTA clusters multicasting V (only 33 clusters of 4 co-reside = 132 SMs:
//    -8%), a 256 x 512 pair tile with one TMEM accumulator (loses the epilogue / MMA overlap:
//    -13%), a dedicated W-storer thread (-4% at K*P = 32).
//
// Warp roles (256 threads): w0 operand TMA producer, w1 MMA issuer + TMEM owner, w2 W TMA
// producer, w3 idle, w4..w7 epilogue (warp w%4 owns TMEM lanes 32*(w%4) .. +31 = tile rows).
// Measured and rejected (kept as compile-time options): two epilogue warpgroups (POS_SFB_EPI=2),
// W slots != 5, BN = 128, KBYTES = 64, L2 evict-first hints.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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
#ifndef POS_SFB_PWSLOTS
#define POS_SFB_PWSLOTS 4
#endif
// The kernel is bound by the W read-modify-write (8 B per element): shared memory goes to W
// prefetch depth (WSLOTS x 16 KB in flight per SM) rather than to operand stages (K*P is small).
constexpr int STAGES = POS_SFB_STAGES;   // operand ring depth
constexpr int WSUB = 32;            // W sub-tile columns (32 fp32 = one 128-byte swizzle row)
constexpr int NSUB = BN / WSUB;     // sub-tiles per tile
constexpr int SWZ = 128;            // swizzle span in bytes (one operand "row" chunk)
#ifndef POS_SFB_KBYTES
#define POS_SFB_KBYTES 128
#endif
constexpr int KBYTES = POS_SFB_KBYTES;   // bytes of K per operand row per stage (BK = KBYTES / elt)
constexpr int A_BYTES = KBYTES * BM;     // per stage: BK rows x BM elements (any dtype)
constexpr int W_BYTES = BM * WSUB * 4;
constexpr int TR = 4;               // tile-index ring depth (dynamic tile scheduler)
#ifndef POS_SFB_PSTAGES
#define POS_SFB_PSTAGES 5   // round 2: 5 stages + 4 W slots beat 4 + 5 at K*P >= 1024 (83 -> 79.5 us, AlexNet fc6)
#endif
// Diagnostics only (never in the shipped build): 1 = no W traffic in the epilogue, 2 = no MMAs,
// 3 = no MMAs and no operand loads.
#ifndef POS_SFB_EXP
#define POS_SFB_EXP 0
#endif
#ifndef POS_SFB_EPI
#define POS_SFB_EPI 1
#endif
#ifndef POS_SFB_PEPI
#define POS_SFB_PEPI 1
#endif
// Epilogue warpgroups (per variant): each owns every EPI-th W sub-tile of the CTA's global
// sub-tile sequence, so one group's TMEM load / smem update overlaps the other's barrier + store.
// Shared-memory layout of one CTA. kPair: CTA-pair kernel (tcgen05 cta_group::2): the pair
// computes a 256 x BN tile, each CTA holds its 128 rows of U and HALF of the tile's V columns,
// so a stage is 2/3 the size and more stages fit — the large-K*P shapes are bound by operand
// bytes in flight, not by W.
template <bool kPair>
struct Lay {
  static constexpr int kStages = kPair ? POS_SFB_PSTAGES : POS_SFB_STAGES;
  static constexpr int kBCols = kPair ? BN / 2 : BN;          // V columns held per CTA
  static constexpr int kBBytes = KBYTES * kBCols;
  static constexpr int kStageBytes = A_BYTES + kBBytes;
  static constexpr int kWSlots = kPair ? POS_SFB_PWSLOTS : POS_SFB_WSLOTS;   // W sub-tile ring depth
  static constexpr int kEpi = kPair ? POS_SFB_PEPI : POS_SFB_EPI;             // epilogue warpgroups
  static constexpr int kThreads = 128 + 128 * kEpi;
  static constexpr int kData = kStages * kStageBytes + kWSlots * W_BYTES;
  static constexpr int kBars = 8 * (2 * kStages + 2 * kWSlots + 4 + 2 * TR) + 16 + 4 * TR;
  static constexpr int kTotal = kData + kBars + 1024;         // + alignment slack
  static constexpr int kTileRows = kPair ? 2 * BM : BM;       // W rows per tile
};
constexpr int STAGE_BYTES = Lay<false>::kStageBytes;
constexpr int SMEM_TOTAL = Lay<false>::kTotal;
constexpr int TMEM_COLS = 2 * BN;

static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
static_assert(Lay<true>::kTotal <= 232448, "shared memory budget (CTA pair)");
// A W slot must always be consumed by the same epilogue group: a group waits on a slot's full
// barrier by phase parity, which is only sound if it consumed the slot's previous phase itself.
static_assert(Lay<false>::kWSlots % Lay<false>::kEpi == 0 && Lay<true>::kWSlots % Lay<true>::kEpi == 0,
              "W slots must be a multiple of the epilogue groups");

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
// D[tmem] (+)= A[smem] * B[smem]^T, one elected thread issues for the whole CTA (kPair: for
// the CTA pair — issued by the even CTA only; the peer's smem is read at the same offsets).
template <bool kTF32, bool kPair>
__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                     uint32_t idesc, uint32_t accumulate) {
#define POS_UMMA(CG, KIND)                                                          \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                   \
               "tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], %1, %2, %3, p;\n}" \
               ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)   \
               : "memory")
  if constexpr (kPair) {
    if constexpr (kTF32) POS_UMMA("2", "tf32"); else POS_UMMA("2", "f16");
  } else {
    if constexpr (kTF32) POS_UMMA("1", "tf32"); else POS_UMMA("1", "f16");
  }
#undef POS_UMMA
}
// mbarrier arrives when all previously issued tcgen05 ops of this thread have completed
// (kPair: on the barrier at this offset in BOTH CTAs of the pair)
template <bool kPair>
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  if constexpr (kPair) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"((uint16_t)0x3)
        : "memory");
  } else {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
  }
}
// ---- cluster (CTA pair) helpers ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// publishes prior shared::cluster stores to the barrier's waiters (tile-ring hand-off only)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar)
               : "memory");
}
// plain arrive on a (possibly remote) barrier: no cluster-scope release fence, which would
// stall the arriving warp on MEMBAR — used where no data is published through the barrier
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// TMA load into this CTA's smem whose completion is signalled on the pair leader's barrier
// (`leader_bar` is a shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar,
                                                 uint32_t dst, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(leader_bar)
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
// N = BN, M = BM (x2 for the CTA pair).
template <bool kTF32, bool kPair = false>
__host__ __device__ constexpr uint32_t instr_desc() {
  return (1u << 4) | ((kTF32 ? 2u : 1u) << 7) | ((kTF32 ? 2u : 1u) << 10) | (1u << 15) |
         (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)((kPair ? 2 * BM : BM) >> 4) << 24);
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
  const unsigned* gsel;   // double-buffered gather: buffer (*gsel - 1) & 1; nullptr = buffer 0
  KTrace trace, group;    // device-side launch trace (off when rec == nullptr)
};

template <bool kTF32, bool kPair>
__global__ void __launch_bounds__(Lay<kPair>::kThreads, 1)
sfb_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA2,
              const __grid_constant__ CUtensorMap tmB2, TileInfo ti, float alpha, int accumulate) {
  using L = Lay<kPair>;
  constexpr int ST = L::kStages;             // operand ring depth
  constexpr int EB = kTF32 ? 4 : 2;          // element bytes
  constexpr int BK = KBYTES / EB;            // k rows per stage (64 bf16 / 32 tf32 at 128 B)
  constexpr int CHUNK = SWZ / EB;            // elements per 128-byte chunk along m / n
  constexpr int UK = 32 / EB;                // UMMA K (16 bf16 / 8 tf32)
  constexpr int BOX_BYTES = BK * SWZ;        // one TMA box: BK rows x 128 B
  constexpr uint32_t IDESC = instr_desc<kTF32, kPair>();
  constexpr int WSLOTS = L::kWSlots, EPI = L::kEpi;
  // epilogue warps that must drain an accumulator before the MMA may overwrite it
  constexpr int kDrainers = 4 * EPI * (kPair ? 2 : 1);
  // tile-ring consumers: (MMA issuer | peer operand producer) + W producer + epilogue, per CTA
  constexpr int kRingConsumers = (2 + 128 * EPI) * (kPair ? 2 : 1);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sW0 = sbase + ST * L::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kData);
  const uint32_t b_full = smem_u32(bars), b_empty = b_full + 8 * ST;
  const uint32_t b_wfull = b_empty + 8 * ST, b_wempty = b_wfull + 8 * WSLOTS;
  const uint32_t b_tfull = b_wempty + 8 * WSLOTS, b_tempty = b_tfull + 16;
  const uint32_t b_rfull = b_tempty + 16, b_rempty = b_rfull + 8 * TR;   // tile-index ring
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 2 * WSLOTS + 4 + 2 * TR);
  volatile int* tile_ring = reinterpret_cast<volatile int*>(tmem_slot + 4);
  const bool dyn = ti.counter != nullptr;
  // CTA pair: the even CTA (rank 0) fetches tiles, issues the MMAs and owns the shared
  // barriers (full, tempty, rempty); each CTA loads and updates its own 128 rows.
  const uint32_t crank = kPair ? cluster_rank() : 0;
  const bool leader = crank == 0;
  const int unit = kPair ? (int)cluster_id_x() : (int)blockIdx.x;   // scheduling unit
  const int nunits = kPair ? (int)nclusters_x() : (int)gridDim.x;
  auto wait_ring = [&](uint32_t bar, uint32_t parity) {
    if constexpr (kPair) mbar_wait_cluster(bar, parity); else mbar_wait(bar, parity);
  };
  // The tile sequence every role walks: static round-robin, or the fetcher's atomic sequence
  // broadcast through the ring (it -> tile, -1 = done). All roles see the same sequence.
  auto tile_of = [&](int it, uint32_t& rphase) -> int {
    if (!dyn) {
      const int t = unit + it * nunits;
      return t < ti.num_tiles ? t : -1;
    }
    const int slot = it % TR;
    wait_ring(b_rfull + 8 * slot, rphase);
    const int t = tile_ring[slot];
    if (kPair) mbar_arrive_remote(map_rank(b_rempty + 8 * slot, 0));
    else mbar_arrive(b_rempty + 8 * slot);
    if (slot == TR - 1) rphase ^= 1;
    return t;
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ktrace_begin(ti.trace);
  ktrace_begin(ti.group);

  if (threadIdx.x == 0) {
    for (int i = 0; i < ST; ++i) { mbar_init(b_full + 8 * i, 1); mbar_init(b_empty + 8 * i, 1); }
    for (int i = 0; i < WSLOTS; ++i) { mbar_init(b_wfull + 8 * i, 1); mbar_init(b_wempty + 8 * i, 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(b_tfull + 8 * i, 1);
      mbar_init(b_tempty + 8 * i, kDrainers);
    }
    for (int i = 0; i < TR; ++i) {
      mbar_init(b_rfull + 8 * i, 1);
      mbar_init(b_rempty + 8 * i, kRingConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // operand maps of the gather buffer this iteration's pack wrote (double buffering)
  const bool second = ti.gsel && ((*reinterpret_cast<const volatile unsigned*>(ti.gsel) - 1u) & 1u);
  const CUtensorMap* mA = second ? &tmA2 : &tmA;
  const CUtensorMap* mB = second ? &tmB2 : &tmB;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(mA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(mB) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
  }
  if (warp == 1) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "n"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (kPair) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== operand TMA producer (+ tile fetcher) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0, rphase = 0;
      for (int it = 0;; ++it) {
        int t;
        if (!dyn) {
          t = unit + it * nunits;
          if (t >= ti.num_tiles) break;
        } else if (kPair && !leader) {
          t = tile_of(it, rphase);
          if (t < 0) break;
        } else {   // fetch the next tile and publish it to the other roles (and the peer CTA)
          const int slot = it % TR;
          wait_ring(b_rempty + 8 * slot, rphase ^ 1);
          t = (int)atomicAdd(ti.counter, 1u);
          if (t >= ti.num_tiles) t = -1;
          tile_ring[slot] = t;
          if constexpr (kPair) {
            st_cluster_u32(map_rank(smem_u32((const void*)&tile_ring[slot]), 1), (uint32_t)t);
            mbar_arrive_cluster(map_rank(b_rfull + 8 * slot, 1));
          }
          mbar_arrive(b_rfull + 8 * slot);
          if (slot == TR - 1) rphase ^= 1;
          if (t < 0) {
            __threadfence();
            if (atomicAdd(ti.counter + 1, 1u) == (unsigned)nunits - 1) {   // last one out resets
              ti.counter[0] = 0;
              ti.counter[1] = 0;
              __threadfence();
            }
            break;
          }
        }
        const int m0 = (t / ti.nb_n) * L::kTileRows + (int)crank * BM;
        const int nb0 = (t % ti.nb_n) * BN + (int)crank * L::kBCols;   // this CTA's V columns
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(b_empty + 8 * stage, phase ^ 1);
          const uint32_t sA = sbase + stage * L::kStageBytes, sB = sA + A_BYTES;
          const int k0 = kb * BK;
          if (POS_SFB_EXP == 3) {   // diagnostic: no operand traffic (and no MMAs)
            if (!kPair || leader) mbar_arrive(b_full + 8 * stage);
          } else if constexpr (kPair) {
            // both CTAs' bytes complete on the leader's full barrier
            const uint32_t full = map_rank(b_full + 8 * stage, 0);
            if (leader) mbar_expect_tx(b_full + 8 * stage, 2 * L::kStageBytes);
#pragma unroll
            for (int c = 0; c < BM / CHUNK; ++c)
              tma_load_2d_pair(mA, full, sA + c * BOX_BYTES, m0 + c * CHUNK, k0);
#pragma unroll
            for (int c = 0; c < L::kBCols / CHUNK; ++c)
              tma_load_2d_pair(mB, full, sB + c * BOX_BYTES, nb0 + c * CHUNK, k0);
          } else {
            const uint32_t full = b_full + 8 * stage;
            mbar_expect_tx(full, L::kStageBytes);
#pragma unroll
            for (int c = 0; c < BM / CHUNK; ++c)
              tma_load_2d(mA, full, sA + c * BOX_BYTES, m0 + c * CHUNK, k0);
#pragma unroll
            for (int c = 0; c < L::kBCols / CHUNK; ++c)
              tma_load_2d(mB, full, sB + c * BOX_BYTES, nb0 + c * CHUNK, k0);
          }
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (single thread; the leader CTA of a pair) ==========
    if (lane == 0 && leader) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase = 0, rphase = 0;
      for (int it = 0;; ++it) {
        const int t = tile_of(it, rphase);
        if (t < 0) break;
        wait_ring(b_tempty + 8 * acc, aphase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(b_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t sA = sbase + stage * L::kStageBytes, sB = sA + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / UK; ++kk) {
            const uint64_t ad = smem_desc<kTF32>(sA + kk * UK * SWZ, BOX_BYTES);
            const uint64_t bd = smem_desc<kTF32>(sB + kk * UK * SWZ, BOX_BYTES);
            if (POS_SFB_EXP != 2 && POS_SFB_EXP != 3) umma<kTF32, kPair>(d_tmem, ad, bd, IDESC, (kb | kk) != 0);
          }
          umma_commit<kPair>(b_empty + 8 * stage);   // frees the smem stage(s) when done
          if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        umma_commit<kPair>(b_tfull + 8 * acc);        // accumulator ready for the epilogue(s)
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
        const int m0 = (t / ti.nb_n) * L::kTileRows + (int)crank * BM, n0 = (t % ti.nb_n) * BN;
        const int nsub = nsub_of(ti.N, n0);
        for (int j = 0; j < nsub; ++j) {
          mbar_wait(b_wempty + 8 * ws, wphase ^ 1);
          const uint32_t wf = b_wfull + 8 * ws;
          if (accumulate && POS_SFB_EXP != 1) {
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
    const int g = (warp - 4) >> 2;            // epilogue warpgroup
    const int et = (threadIdx.x - 128) & 127; // tile row owned by this thread
    const int q = warp & 3;                   // TMEM lane quadrant of this warp
    const uint32_t lane_addr = (uint32_t)(q * 32) << 16;
    constexpr bool kDefer = EPI == 1;         // single group: retire a store one sub-tile later
    int acc = 0;
    uint32_t aphase = 0;
    uint32_t sseq = 0;                        // CTA-wide W sub-tile sequence number
    int pending = -1;                         // slot whose TMA store has not been retired yet
    uint32_t rphase = 0;
    auto release_acc = [&](int a) {           // this warp has drained accumulator a
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair) mbar_arrive_remote(map_rank(b_tempty + 8 * a, 0));
        else mbar_arrive(b_tempty + 8 * a);
      }
    };
    for (int it = 0;; ++it) {
      const int t = tile_of(it, rphase);
      if (t < 0) break;
      const int m0 = (t / ti.nb_n) * L::kTileRows + (int)crank * BM, n0 = (t % ti.nb_n) * BN;
      const int nsub = nsub_of(ti.N, n0);
      // this group's sub-tiles of the tile: j = j0, j0 + EPI, ...; the last one frees TMEM
      const int j0 = (int)((g - (int)(sseq % EPI) + EPI) % EPI);
      const int jlast = j0 < nsub ? j0 + ((nsub - 1 - j0) / EPI) * EPI : -1;
      mbar_wait(b_tfull + 8 * acc, aphase);
      tc_fence_after();
      // A4b fused: the gathered v rows carry a 1.0 in column N, so accumulator column N of the
      // tile holding it is sum_j U[j][m] — the bias gradient of row m
      if (g == 0 && ti.bias && (int64_t)n0 <= ti.N && ti.N < (int64_t)n0 + BN) {
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
      if (jlast < 0) release_acc(acc);        // no sub-tile for this group: release TMEM now
      for (int j = j0; j < nsub; j += EPI) {
        const uint32_t s = sseq + (uint32_t)j;
        const int ws = (int)(s % WSLOTS);
        const uint32_t wphase = (s / WSLOTS) & 1;
        uint32_t r[32];
        tmem_ld32(tmem_base + lane_addr + acc * BN + j * WSUB, r);
        if (j == jlast) release_acc(acc);     // accumulator fully drained by this thread
        mbar_wait(b_wfull + 8 * ws, wphase);
        if (POS_SFB_EXP == 1) {   // diagnostic: no W traffic (TMEM drained, slot recycled)
          named_bar_sync(1 + g, 128);
          if (et == 0) mbar_arrive(b_wempty + 8 * ws);
          continue;
        }
        const uint32_t row = sW0 + ws * W_BYTES + et * SWZ;
        float4 w[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t a = row + ((uint32_t)(c ^ (et & 7)) << 4);   // 128-byte swizzle
          if (accumulate) {
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(w[c].x), "=f"(w[c].y), "=f"(w[c].z), "=f"(w[c].w) : "r"(a));
          } else {
            w[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t a = row + ((uint32_t)(c ^ (et & 7)) << 4);
          w[c].x = fmaf(alpha, __uint_as_float(r[4 * c + 0]), w[c].x);
          w[c].y = fmaf(alpha, __uint_as_float(r[4 * c + 1]), w[c].y);
          w[c].z = fmaf(alpha, __uint_as_float(r[4 * c + 2]), w[c].z);
          w[c].w = fmaf(alpha, __uint_as_float(r[4 * c + 3]), w[c].w);
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(w[c].x),
                       "f"(w[c].y), "f"(w[c].z), "f"(w[c].w)
                       : "memory");
        }
        fence_proxy_async_smem();             // generic-proxy smem writes -> visible to TMA
        named_bar_sync(1 + g, 128);
        if (et == 0) {
          if (POS_SFB_L2HINT)
            tma_store_2d_hint(&tmW, sW0 + ws * W_BYTES, n0 + j * WSUB, m0, policy_evict_first());
          else
            tma_store_2d(&tmW, sW0 + ws * W_BYTES, n0 + j * WSUB, m0);
          bulk_commit();
          if (kDefer) {
            if (pending >= 0) {
              bulk_wait_read<1>();            // the previous store has finished reading smem
              mbar_arrive(b_wempty + 8 * pending);
            }
            pending = ws;
          } else {
            bulk_wait_read<0>();              // the other group keeps the SM busy meanwhile
            mbar_arrive(b_wempty + 8 * ws);
          }
        }
      }
      sseq += (uint32_t)nsub;
      if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (et == 0) bulk_wait_all();
  }

  tc_fence_before();
  if constexpr (kPair) cluster_sync_all(); else __syncthreads();
  ktrace_end(ti.trace);                       // thread 0: every role of this CTA is done
  ktrace_end(ti.group);
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(TMEM_COLS)
                   : "memory");
    else
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

#ifndef POS_SFB_PAIR_KP
#define POS_SFB_PAIR_KP 1024
#endif
// CTA-pair kernel for K*P >= POS_SFB_PAIR_KP (env POS_SFB_PAIR=0|1 forces it off / on,
// POS_SFB_PAIR_KP overrides the threshold; read at plan time).
// cluster_ok = false (the multi-GPU scheduler): no cluster launch unless POS_SFB_PAIR=1 forces it —
// at P = 4 a CUDA-graph step with CTA-pair reconstructions next to the fused cross-GPU kernels
// stalled a rank's factor pack until its peers' watchdogs fired (round 2)
bool use_pair(int64_t KP, bool cluster_ok) {
  if (const char* f = getenv("POS_SFB_PAIR")) {
    if (f[0] == '0') return false;
    if (f[0] == '1') return true;
  }
  if (!cluster_ok) return false;
  int64_t thr = POS_SFB_PAIR_KP;
  if (const char* e = getenv("POS_SFB_PAIR_KP")) thr = atoll(e);
  return KP >= thr;
}

template <bool kTF32, bool kPair>
cudaError_t set_smem_attr() {
  static cudaError_t e = cudaFuncSetAttribute(
      sfb_tc_kernel<kTF32, kPair>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay<kPair>::kTotal);
  return e;
}

// Co-resident CTA pairs of the pair kernel on this device (0 = cannot launch as clusters)
template <bool kTF32>
int max_pairs() {
  static int n = -1;
  if (n < 0) {
    n = 0;
    if (set_smem_attr<kTF32, true>() == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * (unsigned)num_sms());
      cfg.blockDim = dim3(Lay<true>::kThreads);
      cfg.dynamicSmemBytes = Lay<true>::kTotal;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int c = 0;
      if (cudaOccupancyMaxActiveClusters(&c, sfb_tc_kernel<kTF32, true>, &cfg) == cudaSuccess)
        n = c;
      else
        clear_stale_launch_error();
    }
    if (getenv("POS_SFB_VERBOSE"))
      fprintf(stderr, "[poseidon] sfb_tc pair kernel: %d co-resident CTA pairs (%d SMs)\n", n,
              num_sms());
  }
  return n;
}

template <bool kTF32>
bool make_plan_impl(SfbTcPlan* pl, int64_t M, int64_t N, int64_t KP, const void* G, float* W,
                    int64_t ldw, int max_ctas, float* bias, const void* G2, bool cluster_ok) {
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
  if (G2) {
    const uint8_t* g2 = static_cast<const uint8_t*>(G2);
    if (!encode_2d(&pl->tmA2, dt, g2, (uint64_t)M, (uint64_t)KP, (uint64_t)(R * EB), CHUNK, BK,
                   oswz) ||
        !encode_2d(&pl->tmB2, dt, g2 + Mp * EB, (uint64_t)NB, (uint64_t)KP, (uint64_t)(R * EB),
                   CHUNK, BK, oswz))
      return false;
  } else {
    pl->tmA2 = pl->tmA;
    pl->tmB2 = pl->tmB;
  }
  pl->M = M; pl->N = N; pl->KP = KP;
  pl->nb_n = (int)((NB + BN - 1) / BN);
  pl->bias = bias;
  pl->nkb = (int)((KP + BK - 1) / BK);
  pl->tf32 = kTF32;
  int ctas = num_sms();
  if (max_ctas > 0 && max_ctas < ctas) ctas = max_ctas;
  pl->pair = use_pair(KP, cluster_ok) && ctas >= 2 && max_pairs<kTF32>() > 0;
  const int64_t rows = pl->pair ? 2 * BM : BM;
  const int64_t tiles = (int64_t)pl->nb_n * ((M + rows - 1) / rows);
  if (tiles > INT32_MAX) return false;
  pl->num_tiles = (int)tiles;
  // persistent CTAs, or CTA pairs — no more pairs than can be co-resident (a TPC with one
  // usable SM cannot host a pair; a pair that waits for a second wave would be a straggler)
  int units = pl->pair ? std::min(ctas / 2, max_pairs<kTF32>()) : ctas;
  if (units > pl->num_tiles) units = pl->num_tiles;
  pl->grid = pl->pair ? 2 * units : units;
  return true;
}

template <bool kTF32, bool kPair>
cudaError_t launch_plan_impl(const SfbTcPlan& pl, float alpha, int accumulate, cudaStream_t s) {
  clear_stale_launch_error();
  constexpr int smem_bytes = Lay<kPair>::kTotal;
  if (cudaError_t e = set_smem_attr<kTF32, kPair>(); e != cudaSuccess) return e;
  TileInfo ti;
  ti.M = pl.M; ti.N = pl.N; ti.KP = pl.KP;
  ti.nb_n = pl.nb_n; ti.num_tiles = pl.num_tiles; ti.nkb = pl.nkb;
  ti.counter = pl.counter;
  ti.bias = pl.bias;
  ti.gsel = pl.gsel;
  ti.trace = pl.trace;
  if (ti.trace.rec && ti.trace.expected == 0) ti.trace.expected = (unsigned)pl.grid;
  ti.group = pl.group;
  if constexpr (kPair) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)pl.grid);
    cfg.blockDim = dim3(Lay<true>::kThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;   // the CTA pair shares one TPC
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sfb_tc_kernel<kTF32, true>, pl.tmA, pl.tmB, pl.tmW, pl.tmA2,
                              pl.tmB2, ti, alpha, accumulate);
  } else {
    sfb_tc_kernel<kTF32, false><<<pl.grid, Lay<false>::kThreads, smem_bytes, s>>>(
        pl.tmA, pl.tmB, pl.tmW, pl.tmA2, pl.tmB2, ti, alpha, accumulate);
    return cudaGetLastError();
  }
}

}  // namespace

bool sfb_tc_would_pair(int64_t KP, bool cluster_ok) { return use_pair(KP, cluster_ok); }

bool sfb_tc_supported(int64_t N, int64_t ldw, const float* W, const void* G) {
  // TMA stores move whole 16-byte chunks: the last W row chunk must not straddle column N (else
  // the element(s) after N in a strided W would be overwritten) -> N % 4 == 0 as well as ldw.
  return (N % 4) == 0 && (ldw % 4) == 0 && aligned16(W) && aligned16(G) && N >= 1 &&
         get_encode() != nullptr;
}

bool sfb_tc_make_plan(SfbTcPlan* pl, int64_t M, int64_t N, int64_t KP, int32_t dtype,
                      const void* G, float* W, int64_t ldw, int max_ctas, float* bias,
                      const void* G2, bool cluster_ok) {
  if (!sfb_tc_supported(N, ldw, W, G)) return false;
  if (dtype == POS_DT_F32 && f32_ffma()) return false;   // exact-fp32 mode: SIMT FFMA
  if (G2 && !aligned16(G2)) return false;
  if (dtype != POS_DT_BF16)   // TF32, and F32 as the tf32 kind over 3 rows per pair (3xTF32)
    return make_plan_impl<true>(pl, M, N, KP * rows_per_sample(dtype), G, W, ldw, max_ctas, bias,
                                G2, cluster_ok);
  return make_plan_impl<false>(pl, M, N, KP, G, W, ldw, max_ctas, bias, G2, cluster_ok);
}

cudaError_t sfb_tc_launch(const SfbTcPlan& pl, float alpha, int accumulate, cudaStream_t s) {
  if (pl.pair)
    return pl.tf32 ? launch_plan_impl<true, true>(pl, alpha, accumulate, s)
                   : launch_plan_impl<false, true>(pl, alpha, accumulate, s);
  return pl.tf32 ? launch_plan_impl<true, false>(pl, alpha, accumulate, s)
                 : launch_plan_impl<false, false>(pl, alpha, accumulate, s);
}

cudaError_t launch_sfb_tc(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                          int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                          int max_ctas, cudaStream_t s) {
  SfbTcPlan pl;
  if (!sfb_tc_make_plan(&pl, M, N, KP, dtype, G, W, ldw, max_ctas, b)) return cudaErrorInvalidValue;
  return sfb_tc_launch(pl, alpha, accumulate, s);
}


cudaError_t preload_simt_kernels();   // sfb_simt.cu

cudaError_t preload_sfb_kernels() {
  cudaFuncAttributes fa;
  const void* fns[] = {reinterpret_cast<const void*>(sfb_tc_kernel<false, false>),
                       reinterpret_cast<const void*>(sfb_tc_kernel<true, false>),
                       reinterpret_cast<const void*>(sfb_tc_kernel<false, true>),
                       reinterpret_cast<const void*>(sfb_tc_kernel<true, true>)};
  for (const void* f : fns)
    if (cudaError_t e = cudaFuncGetAttributes(&fa, f); e != cudaSuccess) return e;
  // the launch attributes and the co-residency queries the plans use, off the hot path too
  if (cudaError_t e = set_smem_attr<false, false>(); e != cudaSuccess) return e;
  if (cudaError_t e = set_smem_attr<true, false>(); e != cudaSuccess) return e;
  (void)max_pairs<false>();
  (void)max_pairs<true>();
  return preload_simt_kernels();
}

}  // namespace pos
