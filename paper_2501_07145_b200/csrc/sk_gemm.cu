// GEMM-fed FP32 path for channel counts the fused kernel cannot hold in
// registers (d > 16, e.g. BASELINE c4: linear, d = 128).
//
// The cell values of a block of pairs are one dense contraction:
//   rbf:    s(i, j) = <x'_i, y'_j> + n(x'_i) + n(y'_j)   (G = exp2(min(s, 0)))
//   linear: a(i, j) = <dx_i, dy_j>                         (A directly, kernels.py:281)
// with the n-terms folded into K as two extra columns ([x', n_x, 1] . [y', 1, n_y]).
// The tcgen05 3xTF32 GEMM (sk_tcgemm.cu: TMA -> tcgen05.mma -> TMEM, FP32
// accuracy from hi/lo TF32 splits) writes it for a block of x sequences
// against all y into HBM, and `gemm_dp_kernel` streams
// it through the same systolic lane states as the fused kernel (GemmStage
// instead of PointStage): lane q of a segment reads its C columns of two rows
// per step (coalesced 16-lane rows), runs the double difference (rbf) and
// the level recursion, and writes the finished Gram entries. The DP stage is
// HBM-bound by design (4 bytes read per cell); the GEMM is tensor/FP32-bound.
#include <algorithm>
#include <cmath>

#include "sk_gemm.cuh"

namespace sk {
namespace gemm {


// Dense GEMM operand rows: [n][rows][K] float32, split for 3xTF32 into
// hi = rna_tf32(v) and lo = rna_tf32(v - hi) (both written).
//  mode 0 (rbf, x role): [x' (d), n_x, 1, 0...]    mode 1 (rbf, y role): [y', 1, n_y, 0...]
//  mode 2 (linear, both roles): [dx (d), 0...] with dx_0 = 0 (as pack_x/pack_y incr)
// Rows beyond L repeat the last point (rbf) / are zero increments (linear).
__device__ __forceinline__ float rna_tf32(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}
// lo is rounded to TF32 too: the tensor core would otherwise truncate it
// (measured: 4.5x the FP32 SGEMM error, tools/diag_c4_precision.py)
__device__ __forceinline__ void put_split(float *hi, float *lo, int k, float v) {
  const float h = rna_tf32(v);
  hi[k] = h;
  lo[k] = rna_tf32(v - h);
}

__global__ void pack_rows_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                                 int64_t rows, int K, double coord_scale, int mode,
                                 const unsigned long long *__restrict__ mm, int64_t mm_stride,
                                 float *__restrict__ hi, float *__restrict__ lo) {
  const int64_t total = n * rows;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / rows, r = t % rows;
    const double *seq = X + s * L * d;
    const int64_t pt = min(r, L - 1);
    float *dh = hi + t * K, *dl = lo + t * K;
    double nrm = 0.0;
    for (int k = 0; k < d; ++k) {
      double v = seq[pt * d + k];
      if (mode == 2) v = (r >= 1 && r < L) ? v - seq[(pt - 1) * d + k] : 0.0;
      else v -= midrange_of(mm ? mm + s * mm_stride : nullptr, d, k);  // rbf: centring
      const float f = (float)(v * coord_scale);
      put_split(dh, dl, k, f);
      nrm += (double)f * (double)f;
    }
    for (int k = (int)d; k < K; ++k) dh[k] = dl[k] = 0.f;
    if (mode == 0) {
      put_split(dh, dl, (int)d, (float)(-0.5 * nrm));
      put_split(dh, dl, (int)d + 1, 1.f);
    } else if (mode == 1) {
      put_split(dh, dl, (int)d, 1.f);
      put_split(dh, dl, (int)d + 1, (float)(-0.5 * nrm));
    }
  }
}

namespace {

constexpr int RX_MULTI = 8;
constexpr size_t S_BLOCK_BYTES = size_t(2) << 30;  // cell-matrix block budget

struct Plan {
  bool ok = false;
  int C = 8, sw = 0, segs = 0, npanel = 1, nhp = 0, K = 0;
  bool linear = false;
};

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

Plan plan_for(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  Plan pl;
  const int kind = c.static_spec.kind;
  if (c.precision != SK_PREC_FP32 || !c.difference) return pl;
  // linear only. rbf ran here too (the n-terms folded into K) until the
  // extended fuzz found the tensor-core cell values' norm-expansion rounding
  // (|x'|^2 2^-24 near x = y, systematic, multiplied by m at level m) at
  // 1.06x / 1.75x the bar (d = 33, bandwidth ~0.5-0.6), invisible to the
  // certification: rbf with d > 16 takes the float64 row-scan kernel.
  if (kind != SK_LINEAR) return pl;
  if (!fast::fast_orders_supported(c.n_levels, c.order)) return pl;
  if (kind == SK_LINEAR && c.order > 1 && c.normalization != SK_NORM_NONE) return pl;
  if (d < 2 || lx < 2 || ly < 2) return pl;  // d = 1: float64 (see sk_fast.cu plan_for)
  pl.linear = kind == SK_LINEAR;
  pl.K = (int)((pl.linear ? d : d + 2) + 3) / 4 * 4;
  const int C = pl.C = fast::columns_per_lane(c.order);
  if (ly <= 32 * C) {
    pl.sw = next_pow2((int)((ly + C - 1) / C));
  } else {
    pl.sw = 32;
    pl.npanel = (int)((ly + 32 * C - 1) / (32 * C));
    int nch = c.n_levels >= 2 ? c.n_levels - 1 : 0;
    if (c.order > 1)
      for (int m = 1; m < c.n_levels; ++m) nch += std::min(m + 1, (int)c.order) - 1;
    pl.nhp = (2 * nch + 3 + 3) / 4 * 4;
  }
  if ((lx + 1) / 2 < pl.sw) return pl;
  pl.segs = NWARPS * (32 / pl.sw);
  pl.ok = true;
  return pl;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }
int64_t rows_x(int64_t lx) { return 2 * ((lx + 1) / 2); }
int64_t cols_y(const Plan &pl) { return (int64_t)pl.sw * pl.C * pl.npanel; }

double coord_scale(const sk_kernel_config &c) {
  if (c.static_spec.kind == SK_LINEAR) return std::sqrt(c.static_spec.scale);
  return std::sqrt(1.4426950408889634) / c.static_spec.bandwidth;
}

size_t carry_bytes(int64_t lx, const Plan &pl) {
  if (pl.npanel <= 1) return 0;
  return align256((size_t)sm_count() * NWARPS * (RX_MULTI + 2) * ((lx + 1) / 2) * pl.nhp * 4);
}

// x sequences per GEMM block so that the block's cell matrix fits the budget
int64_t block_rows(int64_t nx, int64_t lx, int64_t ny, const Plan &pl) {
  const size_t per_x = (size_t)rows_x(lx) * ny * cols_y(pl) * 4;
  return std::max<int64_t>(1, std::min<int64_t>(nx, (int64_t)(S_BLOCK_BYTES / std::max<size_t>(per_x, 1))));
}

size_t operand_bytes(int64_t n, int64_t rows, const Plan &pl) {  // hi + lo
  return 2 * align256((size_t)n * rows * pl.K * 4);
}

// layout: x operand, y operand, cell-matrix block, carries, midrange codes
size_t gram_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t d, const Plan &pl) {
  const int64_t bx = block_rows(nx, lx, ny, pl);
  return operand_bytes(nx, rows_x(lx), pl) + operand_bytes(ny, cols_y(pl), pl) +
         align256((size_t)bx * rows_x(lx) * ny * cols_y(pl) * 4) + carry_bytes(lx, pl) +
         midrange_bytes(d);
}

size_t self_bytes(int64_t n, int64_t l, int64_t d, const Plan &pl) {
  return operand_bytes(n, rows_x(l), pl) + operand_bytes(n, cols_y(pl), pl) +
         align256((size_t)n * rows_x(l) * cols_y(pl) * 4) + carry_bytes(l, pl) +
         midrange_bytes(n * d);  // per-sequence centres
}

unsigned pack_blocks(int64_t total) {
  return (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
}

// packed hi/lo operand pair of n sequences x rows (hi at `out`, lo after it)
struct Operand {
  float *hi, *lo;
};

Operand carve(void *&cursor, int64_t n, int64_t rows, const Plan &pl) {
  const size_t b = align256((size_t)n * rows * pl.K * 4);
  Operand o{(float *)cursor, (float *)((char *)cursor + b)};
  cursor = (char *)cursor + 2 * b;
  return o;
}

int pack(const double *X, int64_t n, int64_t L, int64_t d, int64_t rows, const Plan &pl,
         const sk_kernel_config &c, bool xrole, const unsigned long long *mm, int64_t mm_stride,
         Operand out, cudaStream_t st) {
  if (n <= 0) return SK_OK;
  const int mode = pl.linear ? 2 : (xrole ? 0 : 1);
  pack_rows_kernel<<<pack_blocks(n * rows), 256, 0, st>>>(X, n, L, d, rows, pl.K, coord_scale(c),
                                                          mode, mm, mm_stride, out.hi, out.lo);
  SK_CHECK_LAUNCH();
  return SK_OK;
}


template <bool LIN>
int launch_dp_lin(const Params &P, int M, int order, cudaStream_t st) {
  using fast::LaneState1;
  using fast::LaneState1D;
  using fast::LaneStateG;
  using S8 = fast::GemmStage<8, LIN>;
  using S4 = fast::GemmStage<4, LIN>;
  if (order == 1 && P.npanel == 1) {  // float64 accumulation (LaneState1D)
    switch (M) {
      case 1: return launch_dp<LaneState1D<S8, 1>, true>(P, st);
      case 2: return launch_dp<LaneState1D<S8, 2>, true>(P, st);
      case 3: return launch_dp<LaneState1D<S8, 3>, true>(P, st);
      case 4: return launch_dp<LaneState1D<S8, 4>, true>(P, st);
      case 5: return launch_dp<LaneState1D<S8, 5>, true>(P, st);
      case 6: return launch_dp<LaneState1D<S8, 6>, true>(P, st);
      case 7: return launch_dp<LaneState1D<S8, 7>, true>(P, st);
      case 8: return launch_dp<LaneState1D<S8, 8>, true>(P, st);
      default: break;
    }
  } else if (order == 1) {
    switch (M) {
      case 1: return launch_dp<LaneState1<S8, 1>>(P, st);
      case 2: return launch_dp<LaneState1<S8, 2>>(P, st);
      case 3: return launch_dp<LaneState1<S8, 3>>(P, st);
      case 4: return launch_dp<LaneState1<S8, 4>>(P, st);
      case 5: return launch_dp<LaneState1<S8, 5>>(P, st);
      case 6: return launch_dp<LaneState1<S8, 6>>(P, st);
      case 7: return launch_dp<LaneState1<S8, 7>>(P, st);
      case 8: return launch_dp<LaneState1<S8, 8>>(P, st);
      default: break;
    }
  } else {
    return launch_dp_geo(P, M, order, LIN, st);
  }
  return fail(SK_ERR_UNSUPPORTED, "gemm path: (n_levels, order) not compiled");
}

Params base_params(const Plan &pl, int64_t lx, float *carry) {
  Params P{};
  P.lx2 = (int)((lx + 1) / 2);
  P.lyp = (int)cols_y(pl);
  P.sw = pl.sw;
  P.segs = pl.segs;
  P.npanel = pl.npanel;
  P.nhp = pl.nhp;
  P.carry = carry;
  P.max_ctas = sm_count();
  P.static_kind = pl.linear ? SK_LINEAR : SK_RBF;  // certification thresholds (write_pair)
  return P;
}

}  // namespace
}  // namespace gemm

bool gemm_supported(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  return gemm::plan_for(lx, ly, d, c).ok;
}

size_t gemm_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                            const sk_kernel_config &c) {
  // ny == 0: self levels of (nx, lx); otherwise the Gram of X (nx, lx) vs Y (ny, ly)
  using namespace gemm;
  if (ny <= 0) {
    const Plan pl = plan_for(lx, lx, d, c);
    return pl.ok ? self_bytes(nx, lx, d, pl) : 0;
  }
  const Plan pl = plan_for(lx, ly, d, c);
  return pl.ok ? gram_bytes(nx, lx, ny, d, pl) : 0;
}

int gemm_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
              int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
              int64_t row_begin, int64_t row_end, const double *diag_x, const double *diag_y,
              double *K, int64_t ldk, double *levels, float *k1buf, void *ws, size_t ws_bytes,
              cudaStream_t st) {
  using namespace gemm;
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  }
  const Plan pl = plan_for(lx, ly, d, c);
  if (!pl.ok) return fail(SK_ERR_UNSUPPORTED, "gemm path does not cover this configuration");
  const size_t need = gram_bytes(nx, lx, ny, d, pl);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  const int64_t rx = rows_x(lx), cy = cols_y(pl), bx = block_rows(nx, lx, ny, pl);
  void *cur = ws;
  const Operand xg = carve(cur, nx, rx, pl);
  const Operand yg = carve(cur, ny, cy, pl);
  float *sblk = (float *)cur;
  float *carry = (float *)((char *)sblk + align256((size_t)bx * rx * ny * cy * 4));
  const unsigned long long *mm = nullptr;
  if (!pl.linear) {
    const int r = midrange(Y, ny, ly, nullptr, 0, 0, d,  // column role (see sk_fast.cu)
                           (unsigned long long *)((char *)carry + carry_bytes(lx, pl)), &mm, st);
    if (r) return r;
  }
  int rc = pack(X, nx, lx, d, rx, pl, c, true, mm, 0, xg, st);
  if (!rc) rc = pack(Y, ny, ly, d, cy, pl, c, false, mm, 0, yg, st);
  if (rc) return rc;
  if (row_end <= row_begin || ny <= 0) return SK_OK;
  Params P = base_params(pl, lx, carry);
  P.nx = nx;
  P.ny = ny;
  P.tiles_y = (ny + pl.segs - 1) / pl.segs;
  P.symmetric = symmetric;
  P.norm = c.normalization;
  P.diag_x = diag_x;
  P.diag_y = symmetric ? diag_x : diag_y;
  P.K = K;
  P.ldk = ldk;
  P.levels = levels;
  P.cert = 1;
  P.k1buf = k1buf;
  P.S = sblk;
  P.s_ld = ny * cy;
  P.s_xstride = rx * ny * cy;
  P.s_ystride = cy;
  const int64_t target = (int64_t)sm_count() * 8;
  for (int64_t b0 = row_begin; b0 < row_end; b0 += bx) {
    const int64_t b1 = std::min(row_end, b0 + bx), rows = b1 - b0;
    // cell matrix of x rows [b0, b1) against all y: (rows*rx) x (ny*cy), row-major
    const int64_t xoff = b0 * rx * pl.K;
    rc = tc_gemm_3xtf32(yg.hi, yg.lo, ny * cy, xg.hi + xoff, xg.lo + xoff, rows * rx, pl.K, sblk,
                        ny * cy, 1, 0, st);
    if (rc) return rc;
    P.x_blk0 = b0;
    P.row_begin = b0;
    P.row_end = b1;
    const int rx_cap = pl.npanel > 1 ? RX_MULTI : 64;
    P.rx = (int)std::max<int64_t>(1, std::min<int64_t>(rx_cap, (rows * P.tiles_y + target - 1) / target));
    P.ntiles = ((rows + P.rx - 1) / P.rx) * P.tiles_y;
    // symmetric K(X): the kernel writes rows >= row_begin of the full matrix;
    // cross: rows relative to the caller's row_begin
    if (!symmetric) {
      P.k1buf = k1buf ? k1buf + 2 * (b0 - row_begin) * ny : nullptr;
      P.K = K ? K + (b0 - row_begin) * ldk : nullptr;
      P.levels = levels ? levels + (b0 - row_begin) * ldk * (c.n_levels + 1) : nullptr;
      P.row_begin = b0;  // write_pair subtracts row_begin
    }
    rc = pl.linear ? launch_dp_lin<true>(P, c.n_levels, c.order, st)
                   : launch_dp_lin<false>(P, c.n_levels, c.order, st);
    if (rc) return rc;
  }
  return SK_OK;
}

int gemm_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                     const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
  using namespace gemm;
  const Plan pl = plan_for(l, l, d, c);
  if (!pl.ok) return fail(SK_ERR_UNSUPPORTED, "gemm path does not cover this configuration");
  if (n <= 0) return SK_OK;
  const size_t need = self_bytes(n, l, d, pl);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  const int64_t rx = rows_x(l), cy = cols_y(pl);
  void *cur = ws;
  const Operand xg = carve(cur, n, rx, pl);
  const Operand yg = carve(cur, n, cy, pl);
  float *sb = (float *)cur;
  float *carry = (float *)((char *)sb + align256((size_t)n * rx * cy * 4));
  unsigned long long *mm = nullptr;
  if (!pl.linear && d <= 1024) {  // self levels: each sequence on its own midrange
    mm = (unsigned long long *)((char *)carry + carry_bytes(l, pl));
    fast::minmax_seq_kernel<<<pack_blocks(n * 32), 256, 0, st>>>(X, n, l, (int)d, mm);
    SK_CHECK_LAUNCH();
  }
  int rc = pack(X, n, l, d, rx, pl, c, true, mm, 2 * d, xg, st);
  if (!rc) rc = pack(X, n, l, d, cy, pl, c, false, mm, 2 * d, yg, st);
  if (rc) return rc;
  // per-sequence cell matrices (pairs (i, i)): batched GEMM, [n][rx][cy]
  rc = tc_gemm_3xtf32(yg.hi, yg.lo, cy, xg.hi, xg.lo, rx, pl.K, sb, cy, n, rx * cy, st);
  if (rc) return rc;
  Params P = base_params(pl, l, carry);
  P.nx = P.ny = n;
  P.tiles_y = (n + pl.segs - 1) / pl.segs;
  P.ntiles = n;  // one tile per sequence (diag mode)
  P.rx = 1;
  P.row_begin = 0;
  P.row_end = n;
  P.diag_mode = 1;
  P.norm = SK_NORM_NONE;
  P.self_out = out;
  // pair (x, y) reads sequence x's own matrix (only x == y is kept)
  P.S = sb;
  P.s_ld = cy;
  P.s_xstride = rx * cy;
  P.s_ystride = 0;
  P.x_blk0 = 0;
  return pl.linear ? launch_dp_lin<true>(P, c.n_levels, c.order, st)
                   : launch_dp_lin<false>(P, c.n_levels, c.order, st);
}

}  // namespace sk
