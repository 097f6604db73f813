// Pure host functions of the C ABI: Algorithm 1, Table 1, the PS shard table, error plumbing,
// and the thin validating wrappers around the kernel launchers.
#include <climits>
#include <cstring>

#include "common.h"

namespace pos {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = '\0'; }

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      return 148;
  }
  return cached;
}

using i128 = __int128;

static bool fits_u64(i128 v) { return v >= 0 && v <= (i128)UINT64_MAX; }

static i128 gcd128(i128 a, i128 b) {
  if (a < 0) a = -a;
  if (b < 0) b = -b;
  while (b) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}

}  // namespace pos

using namespace pos;

extern "C" {

int pos_version(void) { return 200; }

const char* pos_last_error(void) { return g_err; }

// Algorithm 1. Line 7:  2K(P1-1)(M+N) <= 2MN(P1+P2-2)/P2.
// Evaluated exactly as  2K(P1-1)(M+N) * P2 <= 2MN(P1+P2-2)  (reading S4; P2 > 0).
int pos_choose_scheme2(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P1, int32_t P2) {
  clear_error();
  POS_CHECK_ARG(kind == POS_KIND_FC || kind == POS_KIND_DENSE, "unknown layer kind %d", kind);
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && P1 >= 1 && P2 >= 1,
                "M, N, K, P1, P2 must be >= 1 (got %lld %lld %lld %d %d)", (long long)M,
                (long long)N, (long long)K, P1, P2);
  POS_CHECK_ARG(M <= (1LL << 40) && N <= (1LL << 40) && K <= (1LL << 40),
                "M, N, K must be <= 2^40");
  if (kind != POS_KIND_FC) return POS_SCHEME_PS;  // L4: only FC layers can use SFB
  i128 lhs = (i128)2 * K * (P1 - 1) * (i128)(M + N) * P2;
  i128 rhs = (i128)2 * M * N * (i128)(P1 + P2 - 2);
  return lhs <= rhs ? POS_SCHEME_SFB : POS_SCHEME_PS;
}

int pos_choose_scheme(int64_t M, int64_t N, int64_t K, int32_t P) {
  return pos_choose_scheme2(POS_KIND_FC, M, N, K, P, P);
}

// NEXT-3: B200 time model (include/poseidon.h; oracle/cost.py b200_times).
int pos_scheme_times_b200(int64_t M, int64_t N, int64_t K, int32_t P, int32_t factor_bytes,
                          double hbm, double nvl, double tc, double* t_sfb, double* t_ps) {
  clear_error();
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && P >= 1, "M, N, K, P must be >= 1");
  POS_CHECK_ARG(factor_bytes == 2 || factor_bytes == 4, "factor_bytes must be 2 or 4");
  const double m = (double)M, n = (double)N, k = (double)K, p = (double)P;
  const double ihbm = hbm > 0 ? 1.0 / hbm : 0.0, invl = nvl > 0 ? 1.0 / nvl : 0.0,
               itc = tc > 0 ? 1.0 / tc : 0.0;
  const double a_hbm = 8.0 * m * n * ihbm, a_tc = 2.0 * m * n * k * p * itc;
  const double sfb = (p - 1) * k * (m + n) * factor_bytes * invl + (a_hbm > a_tc ? a_hbm : a_tc);
  // multiply before dividing: integer-valued quotients (Alg. 1's ties) stay exact
  const double ps = 8.0 * (p - 1) * m * n / p * invl + 4.0 * m * n * ihbm +
                    12.0 * m * n / p * ihbm;
  if (t_sfb) *t_sfb = sfb;
  if (t_ps) *t_ps = ps;
  return sfb <= ps ? POS_SCHEME_SFB : POS_SCHEME_PS;
}

int pos_scheme_time_adam_b200(int64_t M, int64_t N, int64_t K, int32_t P, int32_t factor_bytes,
                              double hbm, double nvl, double tc, double* t_adam) {
  clear_error();
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && P >= 1, "M, N, K, P must be >= 1");
  POS_CHECK_ARG(factor_bytes == 2 || factor_bytes == 4, "factor_bytes must be 2 or 4");
  POS_CHECK_ARG(t_adam, "NULL output");
  const double m = (double)M, n = (double)N, k = (double)K, p = (double)P;
  const double ihbm = hbm > 0 ? 1.0 / hbm : 0.0, invl = nvl > 0 ? 1.0 / nvl : 0.0,
               itc = tc > 0 ? 1.0 / tc : 0.0;
  const double a_hbm = 8.0 * m * n / p * ihbm, a_tc = 2.0 * m * n * k * itc;
  *t_adam = (p - 1) * k * (m / p + n) * factor_bytes * invl + (a_hbm > a_tc ? a_hbm : a_tc) +
            4.0 * (p - 1) * m * n / p * invl;
  return POS_OK;
}

// Table 1, as exact reduced rationals.
int pos_cost_elems(int32_t scheme, int32_t role, int64_t M, int64_t N, int64_t K, int32_t P1,
                   int32_t P2, uint64_t* num, uint64_t* den) {
  clear_error();
  POS_CHECK_ARG(num && den, "num/den must be non-NULL");
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1 && P1 >= 1 && P2 >= 1, "sizes must be >= 1");
  POS_CHECK_ARG(M <= (1LL << 40) && N <= (1LL << 40) && K <= (1LL << 40), "sizes must be <= 2^40");
  i128 n = 0, d = 1;
  const i128 MN = (i128)M * N, KMN = (i128)K * (M + N);
  switch (scheme) {
    case POS_SCHEME_PS:
      if (role == POS_ROLE_SERVER) { n = 2 * (i128)P1 * MN; d = P2; }
      else if (role == POS_ROLE_WORKER) { n = 2 * MN; }
      else if (role == POS_ROLE_BOTH) { n = 2 * MN * (i128)(P1 + P2 - 2); d = P2; }
      else POS_FAIL(POS_EINVAL, "unknown role %d", role);
      break;
    case POS_SCHEME_SFB:
      if (role == POS_ROLE_WORKER) { n = 2 * (i128)(P1 - 1) * KMN; }
      else if (role == POS_ROLE_SERVER || role == POS_ROLE_BOTH)
        POS_FAIL(POS_EUNSUPPORTED, "SFB cost is N/A for role %d (Table 1)", role);
      else POS_FAIL(POS_EINVAL, "unknown role %d", role);
      break;
    case POS_SCHEME_ADAM:
      if (role == POS_ROLE_SERVER) { n = (i128)P1 * MN + (i128)P1 * KMN; }
      else if (role == POS_ROLE_WORKER) { n = KMN + MN; }
      else if (role == POS_ROLE_BOTH) { n = (i128)(P1 - 1) * (MN + KMN); }
      else POS_FAIL(POS_EINVAL, "unknown role %d", role);
      break;
    default:
      POS_FAIL(POS_EINVAL, "unknown scheme %d", scheme);
  }
  i128 g = gcd128(n, d);
  if (g > 1) { n /= g; d /= g; }
  if (n == 0) d = 1;
  POS_CHECK_ARG(fits_u64(n) && fits_u64(d), "cost overflows uint64");
  *num = (uint64_t)n;
  *den = (uint64_t)d;
  return POS_OK;
}

// PS shard table, reading S9: S = ceil(n / (64 P)) * 64.
int64_t pos_shard_stride(int64_t n, int32_t P) {
  clear_error();
  POS_CHECK_ARG(n >= 1 && P >= 1, "n and P must be >= 1 (got %lld, %d)", (long long)n, P);
  POS_CHECK_ARG(n <= (1LL << 50), "n too large");
  const int64_t g = 64LL * P;
  return (n + g - 1) / g * 64;
}

int pos_shard_range(int64_t n, int32_t P, int32_t r, int64_t* begin, int64_t* end) {
  int64_t S = pos_shard_stride(n, P);
  if (S < 0) return (int)S;
  POS_CHECK_ARG(r >= 0 && r < P, "rank %d out of [0, %d)", r, P);
  POS_CHECK_ARG(begin && end, "begin/end must be non-NULL");
  int64_t lo = (int64_t)r * S, hi = (int64_t)(r + 1) * S;
  *begin = lo < n ? lo : n;
  *end = hi < n ? hi : n;
  return POS_OK;
}

int64_t pos_padded_size(int64_t n, int32_t P) {
  int64_t S = pos_shard_stride(n, P);
  if (S < 0) return S;
  return S * P;
}

int64_t pos_factor_row_elems(int64_t M, int64_t N) {
  clear_error();
  POS_CHECK_ARG(M >= 1 && N >= 1, "M, N must be >= 1");
  return row_elems(M, N);
}

int64_t pos_factor_slot_rows(int64_t K, int32_t dtype) {
  clear_error();
  POS_CHECK_ARG(K >= 0, "K must be >= 0");
  POS_CHECK_ARG(dtype == POS_DT_BF16 || dtype == POS_DT_TF32 || dtype == POS_DT_F32,
                "bad dtype %d", dtype);
  return K * rows_per_sample(dtype);
}

// ---- kernel building blocks ----

int pos_pack_factors(int64_t M, int64_t N, int64_t K, int32_t in_dtype, int32_t dtype,
                     const void* u, const void* v, void* slot, void* stream) {
  clear_error();
  POS_CHECK_ARG(M >= 1 && N >= 1 && K >= 1, "M, N, K must be >= 1");
  POS_CHECK_ARG(in_dtype == POS_IN_BF16 || in_dtype == POS_IN_F32, "bad in_dtype %d", in_dtype);
  POS_CHECK_ARG(dtype == POS_DT_BF16 || dtype == POS_DT_TF32 || dtype == POS_DT_F32,
                "bad dtype %d", dtype);
  POS_CHECK_ARG(u && v && slot, "NULL pointer");
  POS_CHECK_ARG(aligned16(slot), "slot must be 16-byte aligned");
  POS_CUDA_TRY(launch_pack_factors(M, N, K, in_dtype, dtype, u, v, slot, (cudaStream_t)stream));
  return POS_OK;
}

int pos_reconstruct_apply(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                          int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                          void* stream) {
  clear_error();
  return reconstruct_apply(M, N, KP, dtype, G, accumulate, W, ldw, b, alpha, 0,
                           (cudaStream_t)stream);
}

int pos_ps_apply(const float* g, float* W, int64_t count, float alpha, void* stream) {
  clear_error();
  POS_CHECK_ARG(count >= 0, "count must be >= 0");
  POS_CHECK_ARG(count == 0 || (g && W), "NULL pointer");
  if (count == 0) return POS_OK;
  POS_CUDA_TRY(launch_ps_apply(g, W, count, alpha, (cudaStream_t)stream));
  return POS_OK;
}

}  // extern "C"

namespace pos {

int reconstruct_apply(int64_t M, int64_t N, int64_t KP, int32_t dtype, const void* G,
                      int32_t accumulate, float* W, int64_t ldw, float* b, float alpha,
                      int max_ctas, cudaStream_t s) {
  POS_CHECK_ARG(M >= 1 && N >= 1 && KP >= 1, "M, N, KP must be >= 1");
  POS_CHECK_ARG(dtype == POS_DT_BF16 || dtype == POS_DT_TF32 || dtype == POS_DT_F32,
                "bad dtype %d", dtype);
  POS_CHECK_ARG(G && W, "NULL pointer");
  POS_CHECK_ARG(ldw >= N, "ldw %lld < N %lld", (long long)ldw, (long long)N);
  POS_CHECK_ARG(aligned16(G), "G must be 16-byte aligned");
  POS_CHECK_ARG((M * ldw) / ldw == M, "M * ldw overflows");
  cudaError_t e;
  const bool tc = sfb_tc_supported(N, ldw, W, G) && !(dtype == POS_DT_F32 && f32_ffma());
  const int64_t rows = KP * rows_per_sample(dtype);   // 3xTF32 rows for POS_DT_F32
  if (tc) {   // bias fused into the tensor-core epilogue (ones column)
    e = launch_sfb_tc(M, N, KP, dtype, G, accumulate, W, ldw, b, alpha, max_ctas, s);
  } else {
    e = launch_sfb_simt(M, N, rows, dtype, G, accumulate, W, ldw, alpha, s);
  }
  if (e != cudaSuccess)
    POS_FAIL(POS_ECUDA, "reconstruct kernel launch failed: %s", cudaGetErrorString(e));
  if (b && !tc) {
    e = launch_bias_colsum(M, N, rows, dtype, G, accumulate, b, alpha, s);
    if (e != cudaSuccess)
      POS_FAIL(POS_ECUDA, "bias kernel launch failed: %s", cudaGetErrorString(e));
  }
  return POS_OK;
}

}  // namespace pos
