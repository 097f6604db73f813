/*
 * poseidon.h — C ABI of the B200-native Poseidon per-layer gradient synchronisation.
 *
 * Paper: Zhang et al., "Poseidon: An Efficient Communication Architecture for Distributed Deep
 * Learning on GPU Clusters", USENIX ATC'17 (arXiv 1706.03292). Citations below are
 * `PAPER:<line> §<section>` into that text and `SURVEY §8(x)` into
 * SURVEY.md, whose §8 is the hot-path contract this header implements.
 *
 * Conventions (all entry points):
 *  - extern "C", plain pointers and integer sizes; no CUDA, NCCL or torch types. A `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream); an `event` is a cudaEvent_t.
 *  - All sizes are int64_t element counts unless stated. Device pointers are CALLER-OWNED and must
 *    stay valid and unmodified (except by the library) until the operation has completed in
 *    stream order. The library never frees caller memory.
 *  - FC layer notation: W is M x N row-major fp32 with M = out_features and
 *    N = in_features (the nn.Linear.weight layout); b has M entries. Per-sample sufficient factors
 *    (§2.1): u = dL/dy in R^M, v = x in R^N. A worker's K samples are stored as
 *    u: K x M row-major, v: K x N row-major (autograd's grad_output and saved input).
 *  - Update rule: every entry point computes W += alpha * G where G is the summed LOSS gradient
 *    over all P workers (Eq. 2). alpha carries the learning rate, the sign and any
 *    normalisation (readings S5, S6); the library never divides by K or P.
 *  - Errors: synchronous validation returns < 0 (POS_E*) and sets a thread-local message readable
 *    with pos_last_error(). Asynchronous CUDA/NCCL failures are sticky per context and returned by
 *    pos_get_async_error() and by the next call on that context.
 *  - Threading: one host thread drives a context at a time (replaces the paper's CPU thread pool,
 *    PAPER:266 §4.1).
 *  - Determinism: identical inputs give bitwise-identical W on every rank, for both schemes, and
 *    between WFBP and sequential scheduling (no atomics; fixed k order).
 */
#ifndef POSEIDON_H
#define POSEIDON_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pos_ctx pos_ctx;
typedef struct pos_sched pos_sched;
typedef struct pos_loop_fc pos_loop_fc;

/* Communication schemes (§3.2, Table 1). ADAM only for pos_cost_elems. */
enum { POS_SCHEME_PS = 0, POS_SCHEME_SFB = 1, POS_SCHEME_ADAM = 2 };
/* Layer kinds for Algorithm 1: FC is decomposable; DENSE = CONV/BN, "indecomposable" -> PS. */
enum { POS_KIND_FC = 0, POS_KIND_DENSE = 1 };
/* Node roles of Table 1 columns. */
enum { POS_ROLE_SERVER = 0, POS_ROLE_WORKER = 1, POS_ROLE_BOTH = 2 };
/* Factor COMPUTE dtype of the SFB reconstruction (what is gathered and fed to the contraction):
 *   BF16: factors rounded to bf16 (RNE), tcgen05 kind::f16, fp32 accumulate in TMEM.
 *   TF32: factors kept fp32, tcgen05 kind::tf32 (tensor core rounds to tf32), fp32 accumulate.
 *   F32 : factors kept fp32, fp32-accurate: 3xTF32 on tcgen05 kind::tf32 (each pair split into three
 *         tf32 rows, pos_factor_slot_rows), fp32 accumulate; POS_F32_FFMA=1: SIMT FFMA instead. */
enum { POS_DT_BF16 = 0, POS_DT_TF32 = 1, POS_DT_F32 = 2 };
/* Storage dtype of the caller's u / v buffers. */
enum { POS_IN_BF16 = 0, POS_IN_F32 = 1 };
/* Error codes. */
enum {
  POS_OK = 0, POS_EINVAL = -1, POS_ESTATE = -2, POS_ECUDA = -3, POS_ENCCL = -4,
  POS_ENOMEM = -5, POS_EUNSUPPORTED = -6,
  POS_ETIMEOUT = -7   /* a cross-GPU wait exceeded the context's timeout (sticky) */
};
/* Summation order of the PS reduce (pos_set_reduce_order). SWITCH: multimem.ld_reduce, the NVSwitch
 * adds the P gradients (its order) and multimem.st broadcasts the shard; RANK_ORDER: every rank
 * loads the P gradients of its shard from its peers and adds them in rank order 0..P-1 — bitwise
 * reproducible run to run — then multicasts the shard; AUTO (default): at P = 2 rank-order peer loads
 * with plain peer stores (fewest NVLink bytes at P = 2, deterministic), else SWITCH. */
enum { POS_REDUCE_SWITCH = 0, POS_REDUCE_RANK_ORDER = 1, POS_REDUCE_AUTO = 2 };
/* Fault injection (pos_inject_fault; tests of the watchdog):
 *   SKIP_PS  : the given rank does not launch its fused PS kernels (its peers' barriers time out);
 *   SKIP_PACK: loopback only — the given simulated rank does not pack (the flag waits time out). */
enum { POS_FAULT_NONE = 0, POS_FAULT_SKIP_PS = 1, POS_FAULT_SKIP_PACK = 2 };
/* pos_sched_create flags: TIMING = per-unit pack / collective / apply stage events;
 * TIMING_APPLY = only the apply stage (reconstruct-and-apply, shard apply) is bracketed, which
 * adds the fewest graph nodes; SEQUENTIAL = WFBP off (sync after the whole backward). */
enum { POS_SCHED_TIMING = 1, POS_SCHED_SEQUENTIAL = 2, POS_SCHED_TIMING_APPLY = 4,
       POS_SCHED_NO_SYMM = 8 /* keep SFB gather buffers out of symmetric memory (NCCL path) */,
       POS_SCHED_PS_AFTER_SFB = 16 /* P > 1: a dense unit's sync waits for the previously issued
                                      SFB reconstruction instead of overlapping it */,
       POS_SCHED_STATIC_TILES = 32 /* reconstruction tiles in static round-robin order instead of
                                      the dynamic (atomic-counter) tile scheduler */,
       POS_SCHED_TRACE = 64 /* device-side tracing: the apply kernels stamp %globaltimer into device
                               records (pos_sched_trace*) — no event nodes on the streams */ };

/* ABI version (major * 100 + minor): 200 = split factors_ready / weights_free trigger events, watchdog, loopback. */
int pos_version(void);
/* Message of the last < 0 return on this host thread ("" if none). Never NULL. */
const char* pos_last_error(void);

/* ======================================================================================
 * Pure host functions (no context, no GPU).
 * ====================================================================================== */

/* Algorithm 1 BestScheme for an FC layer with P1 = P2 = P (every GPU is both a
 * worker and a PS shard; reading S1). Returns POS_SCHEME_SFB iff
 *     2K(P-1)(M+N) <= 2MN(2P-2)/P,
 * evaluated exactly by 128-bit cross-multiplication (reading S4; tie -> SFB, reading S2; P = 1 ->
 * SFB, reading S8). K is the per-worker batch (reading S3). M, N, K, P >= 1 else POS_EINVAL. */
int pos_choose_scheme(int64_t M, int64_t N, int64_t K, int32_t P);

/* General Algorithm 1 with separate worker count P1 and server count P2 and a layer kind.
 * kind = POS_KIND_DENSE always returns POS_SCHEME_PS. */
int pos_choose_scheme2(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P1, int32_t P2);

/* NEXT-3: B200-calibrated TIME model beside Algorithm 1, in seconds per GPU and
 * iteration for one M x N FC layer with per-GPU batch K on P GPUs:
 *   T_SFB = (P-1) K (M+N) factor_bytes / nvl + max(8 M N / hbm, 2 M N K P / tc)
 *   T_PS  = 2 (P-1)/P * 4 M N / nvl + 4 M N / hbm + 12 M N / (P hbm)
 * (SFB: factors over NVLink, replicated in-place fp32 apply; PS: fp32 reduce-scatter + all-gather,
 * dense dW formation, shard apply.) Bandwidths in bytes/s, tc in flop/s; a value <= 0 drops its
 * terms (hbm <= 0 and tc <= 0 with factor_bytes = 4 reproduce Algorithm 1's decision exactly).
 * Outputs may be NULL. Returns POS_SCHEME_SFB if T_SFB <= T_PS else POS_SCHEME_PS; negative on bad
 * arguments. Oracle: oracle/cost.py b200_times. */
/* The third scheme of Table 1 (Adam: "send SFs to a parameter server shard, then pull back the
 * whole updated parameter matrices") in the same B200 time model, with the layer's rows
 * sharded over the P GPUs (rank s owns M/P rows): every rank pushes u[:, rows(s)] and v to each
 * owner s, the owner reconstructs-and-applies its rows, every rank pulls the other owners' rows:
 *   T_ADAM = (P-1) K (M/P + N) factor_bytes / nvl + max(8 M N / (P hbm), 2 M N K / tc)
 *          + (P-1)/P * 4 M N / nvl
 * Model only (it reports, it does not choose): the fp32 matrix pull costs what the PS all-gather
 * does, so on NVLink it loses to SFB whenever SFB wins and to PS whenever factors outweigh the
 * reduce. Oracle: oracle/cost.py b200_time_adam. Negative on bad arguments. */
int pos_scheme_time_adam_b200(int64_t M, int64_t N, int64_t K, int32_t P, int32_t factor_bytes,
                              double hbm, double nvl, double tc, double* t_adam);
int pos_scheme_times_b200(int64_t M, int64_t N, int64_t K, int32_t P, int32_t factor_bytes,
                          double hbm, double nvl, double tc, double* t_sfb, double* t_ps);
/* Table 1 cost in ELEMENTS as an exact reduced rational num/den (den >= 1).
 * scheme: POS_SCHEME_{PS,SFB,ADAM}; role: POS_ROLE_{SERVER,WORKER,BOTH}. SFB with role SERVER or
 * BOTH is "N/A" in Table 1 -> POS_EUNSUPPORTED. Overflow of uint64 -> POS_EINVAL. */
int pos_cost_elems(int32_t scheme, int32_t role, int64_t M, int64_t N, int64_t K,
                   int32_t P1, int32_t P2, uint64_t* num, uint64_t* den);

/* PS shard table ("partition ... as equally as possible"; reading S9): contiguous
 * shards of stride S = ceil(n / (64 P)) * 64 elements. Returns S (> 0) or < 0 on n < 1 or P < 1. */
int64_t pos_shard_stride(int64_t n, int32_t P);
/* Rank r owns [min(n, r S), min(n, (r+1) S)). */
int pos_shard_range(int64_t n, int32_t P, int32_t r, int64_t* begin, int64_t* end);
/* Elements a caller must allocate for a PS layer's W and grad buffers: P * S. */
int64_t pos_padded_size(int64_t n, int32_t P);
/* Row length (elements) of the library's gathered factor layout for an FC layer:
 * M_pad + N_pad with M_pad = ceil(M/64)*64, N_pad = ceil((N+1)/64)*64 (128-byte aligned rows; column N
 * of the v part is the "ones column" that makes the reconstruction GEMM also produce the bias
 * gradient sum_j u_j, reading S12). */
int64_t pos_factor_row_elems(int64_t M, int64_t N);
/* Gathered rows that K factor pairs occupy in dtype: K for BF16 / TF32, 3K for F32, which runs as
 * 3xTF32 on the tensor cores (reading S16): the pair k is packed as rows k, K+k, 2K+k holding
 * (tf32(u), tf32(v)), (tf32(u), lo(v)), (lo(u), tf32(v)) with lo(x) = tf32(x - tf32(x)); tf32() rounds
 * to nearest, ties away. The contraction over the three rows is u^T v up to the lo(u) lo(v) term and
 * the rounding of lo (relative error ~2^-21 per product). POS_F32_FFMA=1 in the environment (read
 * once per process) selects the exact-fp32 mode instead: K rows, SIMT FFMA reconstruction.
 * Negative on bad arguments. */
int64_t pos_factor_slot_rows(int64_t K, int32_t dtype);

/* ======================================================================================
 * Context: owns the NCCL communicator, a comm stream, a stream pool and scratch buffers.
 * Created on the CURRENT CUDA device of the calling thread.
 * ====================================================================================== */

/* Fill out_128B (128 bytes) with an ncclUniqueId. Call on rank 0, broadcast, then pos_init. */
int pos_get_unique_id(void* out_128B);
/* Collective over `world` processes (one per GPU); blocks until all ranks have joined.
 * With world > 1 the NCCL communicator is capped at POS_NCCL_MAX_CTAS CTAs (env, default 16) and
 * the persistent reconstruction kernel leaves that many SMs (+4) free (POS_SFB_MAX_CTAS env, or
 * pos_set_max_ctas) so collectives are never starved behind it. */
int pos_init(const void* nccl_unique_id_128B, int32_t world, int32_t rank, pos_ctx** out);
/* Single-GPU context simulating P_sim workers (no NCCL): for the pos_sim_* entry points and for
 * P_sim = 1 real single-GPU use. */
int pos_init_local(int32_t P_sim, pos_ctx** out);
/* Destroy the context. CUDA graphs that captured calls on this context must be destroyed first
 * (they hold NCCL resources of its communicator). */
int pos_finalize(pos_ctx* ctx);
int pos_world(const pos_ctx* ctx);
int pos_rank(const pos_ctx* ctx);
/* Sticky asynchronous CUDA/NCCL/watchdog error (POS_OK if none). Does not synchronise: a watchdog
 * expiry is read from a host-mapped error word the kernels write (POS_ETIMEOUT, with the waiting
 * site in pos_last_error()). */
int pos_get_async_error(pos_ctx* ctx);
/* Watchdog budget for every cross-GPU wait inside the library's kernels (entry / exit barriers of
 * the fused PS and gather kernels, gather ready flags): after `ms` milliseconds of spinning the
 * kernel records POS_ETIMEOUT and returns instead of hanging (results of that iteration are
 * undefined; the context is poisoned). 0 = unbounded. Default: env POS_TIMEOUT_MS, else 20000. */
int pos_set_timeout_ms(pos_ctx* ctx, int64_t ms);
/* PS reduce order (POS_REDUCE_*); every rank must set the same. Default POS_REDUCE_AUTO (env
 * POS_REDUCE_ORDER=0|1|2 sets the context default). */
int pos_set_reduce_order(pos_ctx* ctx, int32_t order);
/* Fault injection for tests (POS_FAULT_*); rank = the rank that misbehaves. */
int pos_inject_fault(pos_ctx* ctx, int32_t kind, int32_t rank);
/* Symmetric (NVLink-SHARP multicast) memory, NEXT-1 of SURVEY §8(f). COLLECTIVE: every rank calls
 * with the same size in the same order. The buffer is an NCCL symmetric window on an NVLS
 * multicast object, zero-filled. When a PS layer's W and grad both live in such buffers, its
 * synchronisation (reduce-scatter + shard apply + all-gather) runs as ONE fused kernel:
 * multimem.ld_reduce of the gradient shard through the switch, apply, multimem.st of the fresh W
 * to every replica, between two cross-GPU barriers. The scheduler also places SFB gather buffers
 * there (unless POS_SCHED_NO_SYMM) and multicasts the packed factors into them. Needs world > 1. */
int pos_mem_alloc(pos_ctx* ctx, int64_t bytes, void** out);
int pos_mem_free(pos_ctx* ctx, void* ptr);
/* 1 if [ptr, ptr+bytes) lies inside one pos_mem_alloc buffer, else 0. */
int pos_mem_is_symmetric(pos_ctx* ctx, const void* ptr, int64_t bytes);
/* Cap the number of CTAs of the persistent SFB reconstruction kernel (0 = one per SM). Lets the
 * sync leave SMs to the concurrent backward pass (SURVEY §7 hard part 3). */
int pos_set_max_ctas(pos_ctx* ctx, int32_t max_ctas);

/* ======================================================================================
 * Kernel-level building blocks (stream-ordered, asynchronous). Exposed for tests and callers
 * that bring their own transport.
 * ====================================================================================== */

/* A2 — SFB factor pack ("transformation between SFs and gradients"): write the K rows
 *   slot[k][0 .. M_pad)            = dtype(u[k][0..M)), zero in [M, M_pad)
 *   slot[k][M_pad .. M_pad+N_pad)  = dtype(v[k][0..N)), 1.0 at M_pad+N (ones column), zero after
 * (F32: the 3K rows of pos_factor_slot_rows, each value split as stated there; the ones column
 * splits into 1 / 0 / 1 across the three blocks.)
 * slot: device, pos_factor_slot_rows(K, dtype) * pos_factor_row_elems(M,N) elements of bf16 (dtype
 * BF16) or fp32 (TF32/F32), 16-byte aligned. u, v: device, in_dtype storage, any alignment. */
int pos_pack_factors(int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                     const void* u, const void* v, void* slot, void* stream);

/* A4 + A4b — SFB reconstruct-and-apply (Eq. 2):
 *   W[m][n] = (accumulate ? W[m][n] : 0) + alpha * sum_{j < KP} U[j][m] * V[j][n]
 *   b[m]    = (accumulate ? b[m]    : 0) + alpha * sum_{j < KP} U[j][m]        (if b != NULL)
 * where row j of the gathered buffer G (pos_factor_slot_rows(KP, dtype) rows of
 * pos_factor_row_elems(M,N) elements, packed by pos_pack_factors, worker-major: slot p of K pairs
 * first) holds [u_j | v_j] (F32: the three 3xTF32 rows of each pair, summed). W: device fp32, row
 * stride ldw elements (ldw >= N). Every dtype runs the tcgen05/TMEM/TMA kernel (F32 with the tf32
 * kind over 3*KP rows) when N % 4 == 0, ldw % 4 == 0 and W is 16-byte aligned, else the SIMT FFMA
 * kernel. The k order is fixed, so results are bitwise reproducible. */
int pos_reconstruct_apply(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                          int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                          void* stream);

/* A7 — PS shard apply (PAPER:107 step (2) "apply (+)"): W[i] += alpha * g[i], 0 <= i < count.
 * 16-byte vectorised when both pointers are 16-byte aligned. */
int pos_ps_apply(const float* g, float* W, int64_t count, float alpha, void* stream);

/* ======================================================================================
 * One-shot per-layer synchronisation (stream-ordered on `stream`, returns after enqueue).
 * These share one context workspace: issue them on one stream (or serialise them).
 * ====================================================================================== */

/* SFB: pack this rank's factors, ncclAllGather them over the
 * context's communicator, then W += alpha * U^T V over all K*P samples (and b += alpha*colsum(U)).
 * At world 1 there is no collective. u, v: device, K x M / K x N, in_dtype. */
int pos_sync_layer_sfb(pos_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                       int32_t dtype, const void* u, const void* v, float* W, float* b,
                       float alpha, void* stream);

/* PS for a dense (CONV/BN) layer of n parameters:
 * zero grad[n, P*S) (A5), ncclReduceScatter(sum) in place so rank r holds sum_p g_p on its shard
 * (A6), W[shard r] += alpha * that sum (A7), ncclAllGather(W) in place (A8).
 * grad, W: device fp32 with >= pos_padded_size(n, P) elements, 16-byte aligned; W[n..P*S) is
 * scratch. After completion every rank holds identical W[0..n). */
int pos_sync_layer_ps(pos_ctx* ctx, int64_t n, float* grad, float* W, float alpha, void* stream);

/* PS for an FC layer (scheme forced to PS, or Algorithm 1 chose PS): the local dense gradient
 * G_r = U_r^T V_r (and colsum(U_r) for the bias) is formed by the reconstruction kernel in
 * overwrite mode into grad, then synchronised as a dense layer of n = M*N (+ M if has_bias)
 * parameters laid out [W (M x N row-major) | b (M)]. Wb, grad: >= pos_padded_size(n, P) fp32. */
int pos_sync_layer_fc_ps(pos_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                         int32_t dtype, const void* u, const void* v, float* grad, float* Wb,
                         int32_t has_bias, float alpha, void* stream);

/* Simulated P workers on one GPU (context from pos_init_local(P)). The per-worker inputs are host
 * arrays of P device pointers; the library plays the collective's role by packing every worker's
 * factors into its slot of the gather buffer (SFB), or summing the P gradients in worker order
 * (PS). Results are what every rank would hold after the real synchronisation. */
int pos_sim_sync_layer_sfb(pos_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                           int32_t dtype, const void* const* u, const void* const* v, float* W,
                           float* b, float alpha, void* stream);
int pos_sim_sync_layer_ps(pos_ctx* ctx, int64_t n, const float* const* grads, float* W,
                          float alpha, void* stream);

/* LOOPBACK (single GPU, P = the context's simulated ranks, pos_init_local(P), P <= 16): the SAME
 * kernels as the P > 1 symmetric-memory path, with every cross-GPU address taken from a table of
 * P local replicas and the ranks executed one after the other in stream order (so no barrier is
 * needed). Lets one GPU check the P > 1 kernel bodies (shard reduce -> apply -> broadcast; pack ->
 * slot -> flag publication -> flag wait -> double-buffered reconstruction) against the oracle.
 *
 * PS: for r = 0..P-1, rank r reduces grads[0..P-1] on its shard in rank order, applies
 * W[r][shard] += alpha * sum, and stores the result into the shard of every W[p]. grads[p], W[p]:
 * device fp32, 16-byte aligned, >= pos_padded_size(n, P) elements. */
/* PS over the copy engines (POS_PS_CE, the scheduler's option): the same signal / apply / wait kernels
 * and device-to-device copies as the multi-GPU path, phase by phase over the P replicas (every
 * rank's gradient pieces pushed into its peers' receive slots, every rank's rank-order apply, every
 * fresh shard pushed into every replica, every completion wait). Same arguments and result as
 * pos_loop_sync_layer_ps (bitwise: the same rank-order sum). */
int pos_loop_sync_layer_ps_ce(pos_ctx* ctx, int64_t n, float* const* grads, float* const* W,
                              float alpha, void* stream);
int pos_loop_sync_layer_ps(pos_ctx* ctx, int64_t n, float* const* grads, float* const* W,
                           float alpha, void* stream);
/* SFB: a loopback FC layer with P replicas W[p] (M x N fp32 row-major, 16-byte
 * aligned) and optional b[p] (M). Tensor-core dtypes with N % 4 == 0 use the flag-mode protocol
 * (double-buffered gather buffers per replica, ready flags, device-side buffer selection); other
 * layers the barrier-mode layout. The library owns P gather buffers. */
int pos_loop_fc_create(pos_ctx* ctx, int64_t M, int64_t N, int64_t K, int32_t dtype,
                       float* const* W, float* const* b, pos_loop_fc** out);
/* One iteration: every rank r packs (u[r], v[r]) (K x M / K x N, in_dtype) into its slot of every
 * replica's gather buffer; then every replica waits for the P ready flags and reconstructs
 * W[p] += alpha * U^T V, b[p] += alpha * colsum(U). */
int pos_loop_fc_sync(pos_loop_fc* lf, int32_t in_dtype, const void* const* u, const void* const* v,
                     float alpha, void* stream);
int pos_loop_fc_destroy(pos_loop_fc* lf);

/* ======================================================================================
 * WFBP scheduler (§3.1, Algorithm 2, vector C PAPER:273-275).
 * One record per layer ("syncer"). Per iteration:
 *   pos_sched_begin  -> C := 0
 *   for l = L..1 as backward produces them (Alg. 2 L6-L7):
 *     FC   : pos_sched_factors_ready(l, K, u, v, factors_ready, weights_free)
 *     DENSE: pos_sched_grad_ready(l, grad_ready)
 *   pos_sched_end(consumer)   -> consumer stream waits until all of C is 1 (Alg. 2 L8)
 * A trigger takes CUDA events the caller recorded on its backward stream and enqueues the layer's
 * sync on the library's streams (one comm stream, a pool of apply streams) behind them, so s^l
 * overlaps b^i, i < l. An event must not be re-recorded until its unit is issued (at
 * the trigger of the unit's last layer; at pos_sched_end with POS_SCHED_SEQUENTIAL).
 * Layer indices are 0-based in forward order. Buffers passed at add time must outlive the
 * scheduler. Calls return POS_ESTATE on misuse (trigger twice, end before all triggered,
 * add after begin).
 * Cross-iteration contract (WAR on the library's gather buffers): the triggers of iteration s+1
 * must be stream-ordered after pos_sched_end of iteration s on its consumer stream (or after
 * pos_sched_wait_layer of the same layer) — e.g. the next backward runs on the consumer stream.
 * The flag-mode gather (P > 1, tensor-core dtypes) double-buffers and tolerates one iteration of
 * slack beyond that; the barrier-mode and NCCL gathers do not.
 * ====================================================================================== */
int pos_sched_create(pos_ctx* ctx, int32_t n_layers, int32_t flags, pos_sched** out);
/* FC layer. force_scheme = -1 applies Algorithm 1; else POS_SCHEME_SFB / POS_SCHEME_PS.
 * If the scheme is PS: b must be NULL or W + M*N (one flat [W|b] buffer), and W and grad must
 * have pos_padded_size(M*N (+M), P) elements. Returns the scheme (>= 0) or < 0. */
int pos_sched_add_fc(pos_sched* s, int32_t l, int64_t M, int64_t N, int64_t K, int32_t in_dtype,
                     int32_t dtype, float* W, float* b, float* grad, int32_t force_scheme);
/* DENSE layer of n parameters: W and grad with pos_padded_size(n, P) elements. Returns PS. */
int pos_sched_add_dense(pos_sched* s, int32_t l, int64_t n, float* W, float* grad);
/* A BUCKET of `count` consecutive DENSE layers l_first .. l_first+count-1 stored back to back in
 * one flat buffer (layer l_first+i at offset n[0]+..+n[i-1], no per-layer padding): the paper's
 * fixed-size KV pairs as the PS unit. The bucket (sum n elements; W and grad with
 * pos_padded_size(sum n, P) elements) is synchronised once all its layers have been triggered.
 * Returns PS. */
int pos_sched_add_dense_bucket(pos_sched* s, int32_t l_first, int32_t count, const int64_t* n,
                               float* W, float* grad);
/* Index of the synchronisation unit (layer or bucket) that layer l belongs to. */
int pos_sched_unit_of(pos_sched* s, int32_t l);
int pos_sched_begin(pos_sched* s, float alpha);
/* FC trigger ("(2) ... as long as b_t^l was finished"). rows = the number of sample rows
 * of u (K x M) and v (K x N); it must equal the K registered by pos_sched_add_fc, else POS_EINVAL (a
 * short last batch would make the pack read past u and v: pad it with zero rows, which contribute
 * nothing to U^T V). factors_ready: an event recorded once u (= grad_output) and v (= the saved
 * input) are complete — the pack and the gather wait on it, so they can overlap b^l's grad_input
 * GEMM. weights_free: an event recorded once b^l has finished READING W (after its grad_input
 * GEMM) — the reconstruction, which writes W, waits on it; NULL = factors_ready. u and v must stay
 * valid and unmodified until the layer's sync completes. */
int pos_sched_factors_ready(pos_sched* s, int32_t l, int64_t rows, const void* u, const void* v,
                            void* factors_ready, void* weights_free);
/* DENSE trigger: grad_ready = an event recorded once dW of layer l is complete in its grad buffer
 * (a bucket's sync waits for the events of all its layers). */
int pos_sched_grad_ready(pos_sched* s, int32_t l, void* grad_ready);
/* Per-layer RAW gate: `consumer` waits until layer l's parameters are applied (for f^l of the
 * next iteration; the cross-iteration overlap of PAPER:158). */
int pos_sched_wait_layer(pos_sched* s, int32_t l, void* consumer);
int pos_sched_end(pos_sched* s, void* consumer);
/* Ends the iteration WITHOUT a global wait: every consumer gates itself per layer with
 * pos_sched_wait_layer (f^l of the next iteration waits for s^l only — the cross-iteration overlap
 * of PAPER:158). producer = the backward stream (POS_SCHED_SEQUENTIAL issues the deferred syncs
 * behind it). The WAR contract above then holds per layer through the wait_layer gates. */
int pos_sched_end_layers(pos_sched* s, void* producer);
/* Host wait (after pos_sched_end) until every unit of the last iteration has completed, at most
 * timeout_ms milliseconds (0 = unbounded): POS_ETIMEOUT if not done by then (not sticky: the device
 * work may still finish), the sticky watchdog error at once if a device-side wait expired.
 * Eager iterations only (POS_ESTATE once iterations were captured into CUDA graphs). */
int pos_sched_wait(pos_sched* s, int64_t timeout_ms);
/* Query: the scheme chosen for layer l. */
int pos_sched_scheme(pos_sched* s, int32_t l);
/* With POS_SCHED_TIMING(_APPLY): AVERAGE device milliseconds, over every iteration since the last reset,
 * of layer l's pack, collective(s) (all-gather; or reduce-scatter + all-gather) and apply
 * (reconstruct-and-apply; or shard apply) stages, each bracketed by CUDA events on the stream that
 * runs it. Synchronises on the layer's outstanding iterations. Returns the iteration count (> 0). */
int pos_sched_timing(pos_sched* s, int32_t l, float* pack_ms, float* comm_ms, float* apply_ms);
int pos_sched_timing_reset(pos_sched* s);
/* Tracing, POS_SCHED_TIMING only: the device timeline of the most recent iteration —
 * for unit u (pos_sched_unit_of), out[6u .. 6u+5] = milliseconds of its [start, packed, gathered,
 * apply start, apply end, done] events relative to the first-issued unit's start (-1 = no such
 * stage). Writes at most max_units units; returns the number of units. */
int pos_sched_timeline(pos_sched* s, float* out, int32_t max_units);
/* Device-side tracing (POS_SCHED_TRACE): layer l's unit apply kernel (reconstruct-and-apply; shard
 * apply or fused NVLS PS kernel) — average and last launch duration in microseconds (first CTA
 * start to last CTA end, %globaltimer) and the number of launches since the last reset. Outputs may
 * be NULL. Synchronises the device. */
int pos_sched_trace(pos_sched* s, int32_t l, double* avg_us, double* last_us, int64_t* launches);
/* The last traced launch of layer l's unit apply kernel as absolute %globaltimer stamps (ns; first
 * CTA start, last CTA end) — a timeline of one step without events on the streams. */
int pos_sched_trace_last(pos_sched* s, int32_t l, int64_t* start_ns, int64_t* end_ns);
/* The SPAN of all apply kernels of `scheme` within one step (earliest CTA start of the first to the
 * latest CTA end of the last; they overlap on several streams), averaged over steps. POS_ESTATE if
 * the scheme has no traced kernels (e.g. the SIMT f32 path). */
int pos_sched_trace_span(pos_sched* s, int32_t scheme, double* avg_us, int64_t* steps);
int pos_sched_trace_reset(pos_sched* s);
/* Turn device-side tracing on / off for the iterations issued from now on (between iterations
 * only, else POS_ESTATE). CUDA graphs captured earlier keep the setting they were captured with.
 * Lets a caller time steps untraced and take kernel durations from separately traced steps. The
 * records (pos_sched_trace*) stay readable after tracing is turned off again. */
int pos_sched_set_trace(pos_sched* s, int32_t on);
/* With POS_SCHED_TIMING(_APPLY): the device-time SPAN (earliest apply start to latest apply end)
 * of all units of `scheme` (POS_SCHEME_SFB or POS_SCHEME_PS) within one iteration, averaged over
 * the (up to 4) most recent iterations whose timing events are still live. Reconstructions of
 * different layers may overlap (they alternate between two streams), so this — not the sum of
 * per-layer apply times — is the time the step spends in them. Call it before pos_sched_timing
 * in eager mode (which retires the events). Returns the number of iterations averaged (> 0);
 * POS_ESTATE if none is available. */
int pos_sched_timing_span(pos_sched* s, int32_t scheme, float* span_ms);
int pos_sched_destroy(pos_sched* s);

#ifdef __cplusplus
}
#endif
#endif /* POSEIDON_H */
