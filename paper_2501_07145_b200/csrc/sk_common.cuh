// Shared definitions for the sigkern_b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/sigkern_b200.h"

namespace sk {

// Thread-local error text behind sk_last_error().
void set_error(const std::string &msg);
void clear_error();

#define SK_CHECK_CUDA(expr)                                                        \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::sk::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +       \
                      " at " __FILE__ ":" + std::to_string(__LINE__));             \
      return SK_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

#define SK_CHECK_LAUNCH() SK_CHECK_CUDA(cudaGetLastError())

inline int fail(int code, const std::string &msg) {
  set_error(msg);
  return code;
}

// Number of SMs of the current device (cached per device).
int sm_count();

// ---------------------------------------------------------------------------
// float64 static kernels: static/kernels.py:68-89 (norm-expansion squared
// distance as in kernels.py:256-259 and static/kernels.py:108-114).
// ---------------------------------------------------------------------------
struct StaticF64 {
  int kind;
  int degree;
  double scale, gamma, bandwidth, alpha;
};

__host__ __device__ inline StaticF64 to_static(const sk_static_spec &s) {
  StaticF64 r;
  r.kind = s.kind;
  r.degree = s.degree;
  r.scale = s.scale;
  r.gamma = s.gamma;
  r.bandwidth = s.bandwidth;
  r.alpha = s.alpha;
  return r;
}

__device__ inline double ipow(double b, int e) {
  double r = 1.0;
  for (int k = 0; k < e; ++k) r *= b;
  return r;
}

// Static kernel from the squared distance (stationary kinds) or the inner
// product (linear, polynomial): static/kernels.py:68-89.
__device__ inline double static_from_sq(const StaticF64 &S, double sq) {
  if (sq < 0.0) sq = 0.0;
  const double bw2 = S.bandwidth * S.bandwidth;
  switch (S.kind) {
    case SK_RBF:
      return exp(sq / (-2.0 * bw2));
    case SK_RATIONAL_QUADRATIC:
      return pow(1.0 + sq / (2.0 * S.alpha * bw2), -S.alpha);
    case SK_MATERN12:
      return exp(-(sqrt(sq) / S.bandwidth));
    case SK_MATERN32: {
      const double sr = 1.7320508075688772 * (sqrt(sq) / S.bandwidth);
      return (1.0 + sr) * exp(-sr);
    }
    case SK_MATERN52: {
      const double r = sqrt(sq) / S.bandwidth;
      const double sr = 2.23606797749979 * r;
      return (1.0 + sr + (5.0 / 3.0) * r * r) * exp(-sr);
    }
    default:
      return 0.0;
  }
}
__device__ inline double static_from_inner(const StaticF64 &S, double xy) {
  if (S.kind == SK_LINEAR) return S.scale * xy;
  return pow(S.scale * xy + S.gamma, (double)S.degree);
}

// k(x, y) for two points (stride-1 coordinates).
__device__ inline double static_eval_f64(const StaticF64 &S, const double *x, const double *y,
                                         int d) {
  double xy = 0.0;
  for (int k = 0; k < d; ++k) xy = fma(x[k], y[k], xy);
  if (S.kind == SK_LINEAR || S.kind == SK_POLYNOMIAL) return static_from_inner(S, xy);
  double xx = 0.0, yy = 0.0;
  for (int k = 0; k < d; ++k) {
    xx = fma(x[k], x[k], xx);
    yy = fma(y[k], y[k], yy);
  }
  return static_from_sq(S, xx + yy - 2.0 * xy);
}

// Exact level 1 of a pair (difference=True): the increments telescope,
// sum_ij A_ij = k(x_T, y_T') - k(x_0, y_T') - k(x_T, y_0) + k(x_0, y_0)
// (kernels.py:281 summed over the grid; the level-1 identity of
// test_kernels.py:130-140). x, y are the sequences' float64 points.
__device__ inline double exact_level1(const StaticF64 &S, const double *x, int64_t lx,
                                      const double *y, int64_t ly, int d) {
  if (lx < 2 || ly < 2) return 0.0;
  const double *xT = x + (lx - 1) * d, *yT = y + (ly - 1) * d;
  double s00 = 0.0, s01 = 0.0, s10 = 0.0, s11 = 0.0;  // one pass over the four corners
  if (S.kind == SK_LINEAR || S.kind == SK_POLYNOMIAL) {
    for (int k = 0; k < d; ++k) {
      const double a0 = x[k], a1 = xT[k], b0 = y[k], b1 = yT[k];
      s00 = fma(a0, b0, s00);
      s01 = fma(a0, b1, s01);
      s10 = fma(a1, b0, s10);
      s11 = fma(a1, b1, s11);
    }
    return static_from_inner(S, s11) - static_from_inner(S, s01) - static_from_inner(S, s10) +
           static_from_inner(S, s00);
  }
  for (int k = 0; k < d; ++k) {  // stationary kinds: direct squared distances
    const double a0 = x[k], a1 = xT[k], b0 = y[k], b1 = yT[k];
    s00 = fma(a0 - b0, a0 - b0, s00);
    s01 = fma(a0 - b1, a0 - b1, s01);
    s10 = fma(a1 - b0, a1 - b0, s10);
    s11 = fma(a1 - b1, a1 - b1, s11);
  }
  return static_from_sq(S, s11) - static_from_sq(S, s01) - static_from_sq(S, s10) +
         static_from_sq(S, s00);
}

// FP32 certification thresholds (sk_gram, include/sigkern_b200.h; the
// calibration is in DESIGN.md §4):
//  * realised level-1 noise |k1_fp32 - k1_exact| above the tolerance of its
//    scale (normalised: 1e-5 sqrt(k_1(x,x) k_1(y,y)); unnormalised: 1e-4 |K|;
//    self levels: 1e-5 k_1(x,x)) -> the pair's arithmetic is not trusted;
//  * |K| below CERT_TAU_NORM (normalised) or CERT_TAU_RAW x sum_m |k_m|
//    (unnormalised; linear kind: CERT_TAU_RAW_LINEAR, whose levels are
//    inner products of exact increments) -> cancellation beyond what the FP32
//    level values resolve.
constexpr double CERT_NOISE = 1e-5;
constexpr double CERT_NOISE_RAW = 1e-4;
constexpr double CERT_TAU_NORM = 0.05;
constexpr double CERT_TAU_RAW = 0.01;
constexpr double CERT_TAU_RAW_LINEAR = 0.15;

// ---------------------------------------------------------------------------
// Level-sum epilogue: kernels.py:586-600 (+ _normalize_levelwise 510-516,
// _normalize_global 519-527). lv[0..M] are the pair's level values.
// ---------------------------------------------------------------------------
__device__ inline double finish_entry(const double *lv, int M, int norm, const double *dx,
                                      const double *dy) {
  if (norm == SK_NORM_LEVELWISE) {
    double acc = 0.0;
    for (int m = 0; m <= M; ++m) {
      const double a = dx[m] > 0.0 ? dx[m] : 0.0;
      const double b = dy[m] > 0.0 ? dy[m] : 0.0;
      const double den = sqrt(a * b);
      if (den > 0.0) acc += lv[m] / den;
    }
    return acc / (double)(M + 1);
  }
  double tot = 0.0;
  for (int m = 0; m <= M; ++m) tot += lv[m];
  if (norm == SK_NORM_GLOBAL) {
    double sx = 0.0, sy = 0.0;
    for (int m = 0; m <= M; ++m) {
      sx += dx[m];
      sy += dy[m];
    }
    return tot / sqrt(sx * sy);
  }
  return tot;
}

// ---------------------------------------------------------------------------
// Entry points of the individual translation units.
// ---------------------------------------------------------------------------

// Generic float64 path (any M <= GEN_MAX_LEVELS, p <= GEN_MAX_ORDER, kind, difference).
constexpr int GEN_MAX_LEVELS = 16;
constexpr int GEN_MAX_ORDER = 8;

size_t generic_workspace_bytes(int64_t npairs, int64_t lx, int64_t ly, const sk_kernel_config &c);

int generic_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                 int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
                 int64_t row_begin, int64_t row_end, const double *diag_x,
                 const double *diag_y, double *K, int64_t ldk, double *levels, void *ws,
                 size_t ws_bytes, cudaStream_t st);

int generic_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                        const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                        cudaStream_t st);

size_t generic_levels_dp_workspace_bytes(int64_t batch, int64_t t2, int M, int p);
int generic_levels_from_increments(const double *A, int64_t batch, int64_t t1, int64_t t2,
                                   int M, int p, int per_level, double *out, void *ws,
                                   size_t ws_bytes, cudaStream_t st);

int increment_tensor(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                     int64_t ly, int64_t d, int paired, const sk_static_spec &sp,
                     int difference, double *out, cudaStream_t st);

// Fused FP32 path.
bool fast_supported(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c);
size_t fast_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                            const sk_kernel_config &c);
int fast_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
              int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
              int64_t row_begin, int64_t row_end, const double *diag_x, const double *diag_y,
              double *K, int64_t ldk, double *levels, float *k1buf, void *ws, size_t ws_bytes,
              cudaStream_t st);
int fast_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                     const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                     cudaStream_t st);

// GEMM-fed FP32 path (large d): library GEMM of the cell values + systolic DP.
bool gemm_supported(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c);
size_t gemm_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                            const sk_kernel_config &c);
int gemm_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
              int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
              int64_t row_begin, int64_t row_end, const double *diag_x, const double *diag_y,
              double *K, int64_t ldk, double *levels, float *k1buf, void *ws, size_t ws_bytes,
              cudaStream_t st);
int gemm_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                     const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                     cudaStream_t st);

// tcgen05 3xTF32 GEMM (sk_tcgemm.cu): C[b][n][m] = sum_k A[b][m][k] B[b][n][k]
// from pre-split hi/lo operands (row-major, K a multiple of 4).
int tc_gemm_3xtf32(const float *Ahi, const float *Alo, int64_t Mtot, const float *Bhi,
                   const float *Blo, int64_t Ntot, int K, float *C, int64_t ldc, int64_t batch,
                   int64_t c_bstride, cudaStream_t st);

// Goursat-PDE kernel (algorithm="pde"), float64.
size_t pde_workspace_bytes(int64_t npairs, int64_t ly, int difference);
int pde_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
             int64_t d, int symmetric, const sk_static_spec &sp, int difference,
             int64_t row_begin, int64_t row_end, double *K, int64_t ldk, void *ws,
             size_t ws_bytes, cudaStream_t st);
int pde_self(const double *X, int64_t n, int64_t l, int64_t d, const sk_static_spec &sp,
             int difference, double *out, void *ws, size_t ws_bytes, cudaStream_t st);

// Upper-triangle pairwise distances (median_heuristic), float64.
int pairwise_dist(const double *X, int64_t n, int64_t d, double *out, cudaStream_t st);

// rfsf_exact_gram: static feature maps (sk_features.cu) and lifted level Grams
// on the float64 kernel (sk_generic.cu).
size_t static_features_workspace_bytes(const sk_feature_map &f, int64_t npts);
int static_features(const sk_feature_map &f, const double *X, int64_t npts, int64_t d,
                    double *out, int64_t ld_out, void *ws, size_t ws_bytes, cudaStream_t st);
size_t lifted_workspace_bytes(int64_t npairs, int64_t ly, int M, int order, int difference);
size_t lifted_gram_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int M,
                                   int order, int difference);
int lifted_gram(const double *UX, int64_t nx, int64_t lx, const double *UY, int64_t ny,
                int64_t ly, int64_t width, const int64_t *slot_offsets, int M, int order,
                int difference, int norm, int symmetric, int64_t row_begin, int64_t row_end,
                const double *diag_x, const double *diag_y, double *K, int64_t ldk,
                double *levels, void *ws, size_t ws_bytes, cudaStream_t st);
int lifted_self_levels(const double *UX, int64_t n, int64_t l, int64_t width,
                       const int64_t *slot_offsets, int M, int order, int difference,
                       double *out, void *ws, size_t ws_bytes, cudaStream_t st);

// Centring of translation-invariant static kernels on the FP32 paths: the
// per-channel midrange c = (min + max) / 2 over every point of the column role
// Y (X for K(X) and the self levels) is subtracted from both roles in float64
// before the FP32 rounding (k(x, y) = k(x - c, y - c)); only pairs with x near
// some y have a non-negligible point kernel, so Y's spread bounds |x - c| there.
// The rbf point kernel's norm-expansion exponent carries an absolute FP32
// error of ~|x'|^2 2^-24, so without it accuracy would depend on the data's
// distance from the origin. Min and max are exact in any order, so c is
// deterministic. `mm` holds 2d order-preserving u64 codes (min, then max).
size_t midrange_bytes(int64_t d);
// On success *mm_used is mm, or null when there is nothing to centre (no
// points, or d > 1024).
int midrange(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
             int64_t d, unsigned long long *mm, const unsigned long long **mm_used,
             cudaStream_t st);
__device__ __forceinline__ double ord_dec(unsigned long long u) {
  return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}
// shift of channel k (0 when mm is null)
__device__ __forceinline__ double midrange_of(const unsigned long long *mm, int64_t d, int64_t k) {
  return mm ? 0.5 * (ord_dec(mm[k]) + ord_dec(mm[d + k])) : 0.0;
}

// Float64 fix-ups of the FP32 paths' uncertified results (sk_generic.cu):
// K entries marked NaN by the Gram epilogue, and self levels whose level 0
// was marked NaN by the self-level epilogue. The scratch may alias the FP32
// path's workspace (they run after it in the same stream).
size_t fixup_workspace_bytes(int64_t lx, int64_t ly, const sk_kernel_config &c);
int fp64_fixup(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
               int64_t d, int symmetric, const sk_kernel_config &c, int64_t row_begin,
               int64_t row_end, const double *diag_x, const double *diag_y, const float *k1buf,
               double *K, int64_t ldk, double *levels, void *ws, size_t ws_bytes,
               cudaStream_t st);
int fp64_self_fixup(const double *X, int64_t n, int64_t l, int64_t d, const sk_kernel_config &c,
                    double *out, void *ws, size_t ws_bytes, cudaStream_t st);

// Certification buffer at the start of an FP32 Gram's workspace (the path's
// own workspace follows): per entry a float2 (FP32 level 1, sum_m |k_m|).
inline size_t k1buf_bytes(int64_t nx, int64_t ny, int /*norm*/) {
  return ((size_t)nx * ny * 8 + 255) & ~(size_t)255;
}

// Order-1 float64 recursion with one CTA per pair (sk_rowscan.cu): the
// float64 Gram / self levels for rows of >= 32 increments, and the FP32
// certification's exact-level-1 pass + float64 redo of flagged entries.
bool warp_gram_ok(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c);
bool rowscan_supported(int64_t lx, int64_t ly, const sk_kernel_config &c);
size_t rowscan_workspace_bytes(int64_t npairs, int64_t lx, int64_t ly, const sk_kernel_config &c);
// mode 0 rect, 1 symmetric, 2 self levels (self_out)
int rowscan_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                 int64_t ly, int64_t d, int mode, const sk_kernel_config &c, int64_t row_begin,
                 int64_t row_end, const double *diag_x, const double *diag_y, double *K,
                 int64_t ldk, double *levels, double *self_out, void *ws, size_t ws_bytes,
                 cudaStream_t st);
size_t cert_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                            const sk_kernel_config &c);
int cert_fixup(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
               int64_t d, int symmetric, const sk_kernel_config &c, int64_t row_begin,
               int64_t row_end, const double *diag_x, const double *diag_y, const float *k1buf,
               double *K, int64_t ldk, double *levels, void *ws, size_t ws_bytes,
               cudaStream_t st);
int cert_self_fixup(const double *X, int64_t n, int64_t l, int64_t d, const sk_kernel_config &c,
                    double *out, void *ws, size_t ws_bytes, cudaStream_t st);

// Path selection: 1 fused, 2 GEMM-fed, 0 float64.
inline int path_of(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  if (fast_supported(lx, ly, d, c)) return 1;
  if (gemm_supported(lx, ly, d, c)) return 2;
  return 0;
}

}  // namespace sk
