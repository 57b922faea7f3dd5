// Host side of the fused FP32 path: shape planning, input packing and launch.
#include <algorithm>
#include <cmath>

#include "sk_fast.cuh"

namespace sk {
namespace fast {

// Packed value of channel k at packed index r of one sequence, and whether
// the slot is a dummy (point kernel 0). mode: 0 points (rows beyond L repeat
// the last point: zero increments); 1 increments x_r - x_{r-1} (0 for r = 0
// and beyond L); 2/3 difference=False (rbf / linear), x role: row 0 and rows
// beyond L are dummies, row r holds point r-1; y role: point r, dummies
// beyond L.
// shift: the midrange centring of the point modes (0 and 2; sk_common.cuh).
__device__ __forceinline__ double packed_coord(const double *__restrict__ seq, int64_t L,
                                               int64_t d, int64_t r, int k, int mode,
                                               bool xrole, double shift, bool &dummy) {
  dummy = false;
  if (mode >= 2) {
    const int64_t pt = xrole ? r - 1 : r;
    if (pt < 0 || pt >= L) {
      dummy = true;
      return 0.0;
    }
    return mode == 2 ? seq[pt * d + k] - shift : seq[pt * d + k];
  }
  const int64_t pt = min(r, L - 1);
  double v = seq[pt * d + k];
  if (mode == 1) v = (r >= 1 && r < L) ? v - seq[(pt - 1) * d + k] : 0.0;
  else v -= shift;
  return v;
}

__device__ __forceinline__ unsigned long long ord_enc(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Per-channel min/max codes of `total` values laid out [..][d]. blockDim is a
// multiple of d, and so is the grid stride: every thread sees one channel.
__global__ void minmax_kernel(const double *__restrict__ X, int64_t total, int d,
                              unsigned long long *__restrict__ mm) {
  extern __shared__ unsigned long long red[];  // [2][blockDim]
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long u = ord_enc(X[t]);
    lo = u < lo ? u : lo;
    hi = u > hi ? u : hi;
  }
  red[threadIdx.x] = lo;
  red[blockDim.x + threadIdx.x] = hi;
  __syncthreads();
  if (threadIdx.x < d) {
    for (int t = threadIdx.x + d; t < (int)blockDim.x; t += d) {
      lo = red[t] < lo ? red[t] : lo;
      hi = red[blockDim.x + t] > hi ? red[blockDim.x + t] : hi;
    }
    atomicMin(mm + threadIdx.x, lo);
    atomicMax(mm + d + threadIdx.x, hi);
  }
}

// Per-sequence min/max codes (the self-level passes: every sequence centred
// on its own midrange, so self levels do not depend on the batch): one warp
// per sequence, mm[s][0..d) min and [d..2d) max.
__global__ void minmax_seq_kernel(const double *__restrict__ X, int64_t n, int64_t L, int d,
                                  unsigned long long *__restrict__ mm) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = w0; s < n; s += nw) {
    const double *seq = X + s * L * d;
    for (int k = 0; k < d; ++k) {
      unsigned long long lo = ~0ull, hi = 0ull;
      for (int64_t r = lane; r < L; r += 32) {
        const unsigned long long u = ord_enc(seq[r * d + k]);
        lo = u < lo ? u : lo;
        hi = u > hi ? u : hi;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
        lo = a < lo ? a : lo;
        hi = b > hi ? b : hi;
      }
      if (lane == 0) {
        mm[s * 2 * d + k] = lo;
        mm[s * 2 * d + d + k] = hi;
      }
    }
  }
}

// n-term slot: -|x'|^2/2 for the rbf modes (-1e30 for dummies), 0 for linear
__device__ __forceinline__ float nterm(int mode, double nrm, bool dummy) {
  if (mode == 1 || mode == 3) return 0.f;
  return dummy ? -1e30f : (float)(-0.5 * nrm);
}

__global__ void pack_y_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                              int64_t Lp, int D, double coord_scale, int mode,
                              const unsigned long long *__restrict__ mm, int64_t mm_stride,
                              float *__restrict__ out) {
  const int YP = y_stride(D);
  const int64_t total = n * Lp;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / Lp;
    const double *seq = X + s * L * d;
    const unsigned long long *ms = mm ? mm + s * mm_stride : nullptr;
    float *dst = out + t * YP;
    double nrm = 0.0;
    bool dummy = false;
    for (int k = 0; k < D; ++k) {
      const float v =
          (k < d) ? (float)(packed_coord(seq, L, d, t % Lp, k, mode, false, midrange_of(ms, d, k),
                                         dummy) * coord_scale)
                  : 0.f;
      dst[k] = v;
      nrm += (double)v * (double)v;  // n-term from the rounded coordinates
    }
    dst[D] = nterm(mode, nrm, dummy);
    for (int k = D + 1; k < YP; ++k) dst[k] = 0.f;
  }
}

__global__ void pack_x_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                              int64_t Lp2, int D, double coord_scale, int mode,
                              const unsigned long long *__restrict__ mm, int64_t mm_stride,
                              float *__restrict__ out) {
  const int XP = x_stride(D);
  const int64_t total = n * Lp2 * 2;  // one thread per (sequence, row)
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / (2 * Lp2);
    const int64_t r = t % (2 * Lp2);
    const int half = (int)(r & 1);
    const double *seq = X + s * L * d;
    const unsigned long long *ms = mm ? mm + s * mm_stride : nullptr;
    float *dst = out + (s * Lp2 + (r >> 1)) * XP;
    double nrm = 0.0;
    bool dummy = false;
    for (int k = 0; k < D; ++k) {
      const float v =
          (k < d) ? (float)(packed_coord(seq, L, d, r, k, mode, true, midrange_of(ms, d, k), dummy) *
                            coord_scale)
                  : 0.f;
      dst[2 * k + half] = v;
      nrm += (double)v * (double)v;
    }
    dst[2 * D + half] = nterm(mode, nrm, dummy);
    dst[2 * D + 2 + half] = 0.f;
  }
}

namespace {

#ifndef SK_RX_MULTI
#define SK_RX_MULTI 8
#endif
constexpr int RX_MULTI = SK_RX_MULTI;  // x sequences per tile when the carry buffer is in use

struct Plan {
  bool ok = false;
  int D = 0, C = 8, sw = 0, segs = 0, npanel = 1, nhp = 0;
  bool linear = false;
  bool nodiff = false;  // difference=False: the x role carries a dummy row 0
  int variant = 0;  // 0 rbf, 1 linear, 2 stationary kinds (matern*, rational quadratic),
                    // 3 rbf difference=False
};

bool stationary_kind(int kind) {
  return kind == SK_MATERN12 || kind == SK_MATERN32 || kind == SK_MATERN52 ||
         kind == SK_RATIONAL_QUADRATIC;
}

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

constexpr size_t SMEM_LIMIT = 200 * 1024;

// x rows per sequence: L points, plus the dummy row 0 when difference=False
int64_t pairs_of(int64_t lx, const Plan &pl) { return (lx + (pl.nodiff ? 1 : 0) + 1) / 2; }

Plan plan_for(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  Plan pl;
  const int kind = c.static_spec.kind;
  if (c.precision != SK_PREC_FP32) return pl;
  const bool stat = stationary_kind(kind);
  // polynomial: float64 kernels. The FP32 recursion loses it to cancellation
  // INSIDE the high levels (terms ~(scale <x,y> + gamma)^degree, level sums
  // orders of magnitude below them), which neither certification rule sees:
  // a 1500-case sweep measured up to 12x the 1e-4 bar
  if (kind == SK_POLYNOMIAL) return pl;
  pl.nodiff = !c.difference;
  if (pl.nodiff && stat) return pl;  // not compiled
  if (!fast_orders_supported(c.n_levels, c.order)) return pl;
  // Normalised linear kernels of order > 1 are sensitive to the FP32
  // accumulation of the increment inner products (measured 1.6-2.1e-5 vs the
  // 1e-5 bar, also in a float64-recursion emulation): float64 kernel.
  if (kind == SK_LINEAR && c.order > 1 && c.normalization != SK_NORM_NONE) return pl;
  const int64_t lmin = c.difference ? 2 : 1;  // difference=False: one point is one cell
  // d = 1: one-dimensional paths are cancellation-dominated (level m is
  // (x_T - x_0)^m/m! from terms of size (sum |dx|)^m/m!); the FP32 sweep
  // measured 1.7e-5 normalised: float64 kernel
  if (d < 2 || d > 16 || lx < lmin || ly < lmin) return pl;
  // d = 2 at general order (non-linear kinds, differenced): the high levels of
  // nearly planar increments cancel internally, which the certification does
  // not see; tools/path_sweep.py measured up to 4.8x the levelwise bar there
  // and <= 0.64x at d >= 3: float64 kernel
  if (d == 2 && c.order > 1 && c.n_levels > 1 && kind != SK_LINEAR && c.difference) return pl;
  pl.D = d <= 4 ? 4 : (d <= 8 ? 8 : 16);
  const int C = pl.C = columns_per_lane(c.order);
  if (ly <= 32 * C) {
    pl.sw = next_pow2((int)((ly + C - 1) / C));
  } else {  // sequential 32*C-column panels with chain carries through HBM/L2
    pl.sw = 32;
    pl.npanel = (int)((ly + 32 * C - 1) / (32 * C));
    // chain values per row: p = 1: levels 1..M-1; general p: S and E chains
    int nch = c.n_levels >= 2 ? c.n_levels - 1 : 0;
    if (c.order > 1)
      for (int m = 1; m < c.n_levels; ++m) nch += std::min(m + 1, (int)c.order) - 1;
    pl.nhp = (2 * nch + 3 + 3) / 4 * 4;
  }
  const int64_t lx2 = pairs_of(lx, pl);
  if (lx2 < pl.sw) return pl;
  // + one pad record: the row prefetch may read one record past the last slot
  if (((size_t)NSLOT * lx2 + 1) * x_stride(pl.D) * sizeof(float) > SMEM_LIMIT) return pl;
  pl.segs = NWARPS * (32 / pl.sw);
  pl.linear = kind == SK_LINEAR;
  pl.variant = pl.linear ? 1 : (stat ? 2 : (pl.nodiff ? 3 : 0));
  pl.ok = true;
  return pl;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int lyp_of(const Plan &pl) { return pl.sw * pl.C * pl.npanel; }

size_t carry_bytes(int64_t lx, const Plan &pl) {
  if (pl.npanel <= 1) return 0;
  return align256((size_t)sm_count() * NWARPS * (RX_MULTI + 2) * pairs_of(lx, pl) * pl.nhp *
                  sizeof(float));
}

size_t x_bytes(int64_t n, int64_t lx, const Plan &pl) {
  return align256((size_t)n * pairs_of(lx, pl) * x_stride(pl.D) * sizeof(float));
}
size_t y_bytes(int64_t n, const Plan &pl) {
  return align256((size_t)n * lyp_of(pl) * y_stride(pl.D) * sizeof(float));
}
size_t roles_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t d, const Plan &pl,
                   bool self_pass = false) {
  return x_bytes(nx, lx, pl) + y_bytes(ny, pl) + carry_bytes(lx, pl) +
         midrange_bytes(self_pass ? nx * d : d);
}

double coord_scale(const sk_kernel_config &c) {
  if (c.static_spec.kind == SK_LINEAR) return std::sqrt(c.static_spec.scale);
  if (stationary_kind(c.static_spec.kind)) return 1.0 / c.static_spec.bandwidth;  // r = |x'-y'|
  // G = exp(-|x-y|^2 / (2 bw^2)) = exp2(-|x'-y'|^2 / 2) with x' = x sqrt(log2 e) / bw
  return std::sqrt(1.4426950408889634) / c.static_spec.bandwidth;
}

unsigned pack_blocks(int64_t total) {
  return (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
}

int launch(const Params &P, const Plan &pl, int M, int order, cudaStream_t st) {
  // + one pad record: the row prefetch may read one record past the last slot
  const size_t smem = ((size_t)NSLOT * P.lx2 + 1) * x_stride(pl.D) * sizeof(float);
  switch (pl.D) {
    case 4:
      return launch_d4(P, M, order, pl.variant, smem, st);
    case 8:
      return launch_d8(P, M, order, pl.variant, smem, st);
    case 16:
      return launch_d16(P, M, order, pl.variant, smem, st);
    default:
      return fail(SK_ERR_UNSUPPORTED, "fast path: unsupported channel padding");
  }
}

// Pack both roles into the workspace: x row pairs [nx][lx2], y columns
// [ny][lyp], then the carry buffer.
struct Packed {
  const float *xs, *ys;
  int lx2, lyp;
  float *carry;
};

// self_pass: both roles are X and every sequence is centred on its own midrange
int pack_roles(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
               int64_t ly, int64_t d, const Plan &pl, const sk_kernel_config &c, void *ws,
               size_t ws_bytes, cudaStream_t st, Packed &out, bool self_pass = false) {
  const size_t need = roles_bytes(nx, lx, ny, d, pl, self_pass);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
  const size_t bx = x_bytes(nx, lx, pl), by = y_bytes(ny, pl);
  float *xsb = (float *)ws;
  float *ysb = (float *)((char *)ws + bx);
  const int64_t lx2 = pairs_of(lx, pl), lyp = lyp_of(pl);
  const double cs = coord_scale(c);
  // packing mode (pack_x/pack_y): linear: A = <dx, dy> directly from increments
  const int incr = pl.nodiff ? (pl.linear ? 3 : 2) : (pl.linear ? 1 : 0);
  // translation-invariant kinds: midrange centring (sk_common.cuh)
  const unsigned long long *mm = nullptr;
  int64_t mm_stride = 0;
  if (!pl.linear) {
    unsigned long long *mmb =
        (unsigned long long *)((char *)ws + bx + by + carry_bytes(lx, pl));
    if (self_pass) {
      // self levels: each sequence on its own midrange (batch-independent)
      if (d <= 1024 && nx > 0) {
        minmax_seq_kernel<<<pack_blocks(nx * 32), 256, 0, st>>>(X, nx, lx, (int)d, mmb);
        SK_CHECK_LAUNCH();
        mm = mmb;
        mm_stride = 2 * d;
      }
    } else {
      // Gram: centre of the column role only, so rows of K(X, Y) are the Gram
      // of those rows bit for bit
      const int rc = midrange(Y, ny, ly, nullptr, 0, 0, d, mmb, &mm, st);
      if (rc) return rc;
    }
  }
  if (nx > 0) {
    pack_x_kernel<<<pack_blocks(nx * lx2 * 2), 256, 0, st>>>(X, nx, lx, d, lx2, pl.D, cs, incr,
                                                             mm, mm_stride, xsb);
    SK_CHECK_LAUNCH();
  }
  if (ny > 0) {
    pack_y_kernel<<<pack_blocks(ny * lyp), 256, 0, st>>>(Y, ny, ly, d, lyp, pl.D, cs, incr,
                                                         mm, mm_stride, ysb);
    SK_CHECK_LAUNCH();
  }
  out.xs = xsb;
  out.ys = ysb;
  out.lx2 = (int)lx2;
  out.lyp = (int)lyp;
  out.carry = (float *)((char *)ws + bx + by);
  return SK_OK;
}

Params base_params(const Plan &pl, const Packed &pk, const sk_kernel_config &c) {
  Params P{};
  P.static_kind = c.static_spec.kind;
  P.rq_alpha = (float)c.static_spec.alpha;
  P.xs = pk.xs;
  P.ys = pk.ys;
  P.lx2 = pk.lx2;
  P.lyp = pk.lyp;
  P.sw = pl.sw;
  P.segs = pl.segs;
  P.npanel = pl.npanel;
  P.nhp = pl.nhp;
  P.carry = pk.carry;
  P.max_ctas = sm_count();
  return P;
}

}  // namespace
}  // namespace fast

bool fast_supported(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  return fast::plan_for(lx, ly, d, c).ok;
}

size_t fast_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                            const sk_kernel_config &c) {
  // ny == 0: self levels of (nx, lx); otherwise the Gram of X (nx, lx) vs Y (ny, ly)
  using namespace fast;
  const Plan pl = ny > 0 ? plan_for(lx, ly, d, c) : plan_for(lx, lx, d, c);
  if (!pl.ok) return 0;
  return roles_bytes(nx, lx, ny > 0 ? ny : nx, d, pl, ny <= 0);
}

size_t midrange_bytes(int64_t d) { return (2 * (size_t)d * 8 + 255) & ~(size_t)255; }

int midrange(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
             int64_t d, unsigned long long *mm, const unsigned long long **mm_used,
             cudaStream_t st) {
  const int64_t tx = nx * lx * d, ty = Y ? ny * ly * d : 0;
  *mm_used = nullptr;
  if (d < 1 || d > 1024 || tx + ty == 0) return SK_OK;
  SK_CHECK_CUDA(cudaMemsetAsync(mm, 0xff, (size_t)d * 8, st));
  SK_CHECK_CUDA(cudaMemsetAsync(mm + d, 0, (size_t)d * 8, st));
  const int bd = (int)(d * std::max<int64_t>(1, 256 / d));
  const size_t sh = 2 * (size_t)bd * 8;
  for (int r = 0; r < 2; ++r) {
    const double *src = r ? Y : X;
    const int64_t tot = r ? ty : tx;
    if (tot == 0) continue;
    const unsigned g = (unsigned)std::min<int64_t>((tot + bd - 1) / bd, (int64_t)sm_count() * 4);
    fast::minmax_kernel<<<g, bd, sh, st>>>(src, tot, (int)d, mm);
    SK_CHECK_LAUNCH();
  }
  *mm_used = mm;
  return SK_OK;
}

int fast_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
              int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
              int64_t row_begin, int64_t row_end, const double *diag_x, const double *diag_y,
              double *K, int64_t ldk, double *levels, float *k1buf, void *ws, size_t ws_bytes,
              cudaStream_t st) {
  using namespace fast;
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  }
  const Plan pl = plan_for(lx, ly, d, c);
  if (!pl.ok) return fail(SK_ERR_UNSUPPORTED, "fast path does not cover this configuration");
  Packed pk{};
  int rc = pack_roles(X, nx, lx, Y, ny, ly, d, pl, c, ws, ws_bytes, st, pk);
  if (rc) return rc;
  Params P = base_params(pl, pk, c);
  P.nx = nx;
  P.ny = ny;
  P.tiles_y = (ny + pl.segs - 1) / pl.segs;
  const int64_t rows = row_end - row_begin;
  if (rows <= 0 || ny <= 0) return SK_OK;
  const int64_t target = (int64_t)sm_count() * 8;
  const int rx_cap = pl.npanel > 1 ? RX_MULTI : 64;
  P.rx = (int)std::max<int64_t>(1, std::min<int64_t>(rx_cap, (rows * P.tiles_y + target - 1) / target));
  P.ntiles = ((rows + P.rx - 1) / P.rx) * P.tiles_y;
  P.row_begin = row_begin;
  P.row_end = row_end;
  P.symmetric = symmetric;
  P.diag_mode = 0;
  P.norm = c.normalization;
  P.diag_x = diag_x;
  P.diag_y = symmetric ? diag_x : diag_y;
  P.K = K;
  P.ldk = ldk;
  P.levels = levels;
  P.cert = 1;
  P.k1buf = k1buf;
  return launch(P, pl, c.n_levels, c.order, st);
}

int fast_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                     const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
  using namespace fast;
  const Plan pl = plan_for(l, l, d, c);
  if (!pl.ok) return fail(SK_ERR_UNSUPPORTED, "fast path does not cover this configuration");
  if (n <= 0) return SK_OK;
  Packed pk{};
  int rc = pack_roles(X, n, l, X, n, l, d, pl, c, ws, ws_bytes, st, pk, true);
  if (rc) return rc;
  // each CTA evaluates its segments' y against the same sequences as x and
  // keeps the diagonal: the same kernel and arithmetic as the Gram's diagonal
  Params P = base_params(pl, pk, c);
  P.nx = P.ny = n;
  P.tiles_y = (n + pl.segs - 1) / pl.segs;
  P.ntiles = n;  // one tile per sequence (diag mode)
  P.rx = 1;
  P.row_begin = 0;
  P.row_end = n;
  P.diag_mode = 1;
  P.norm = SK_NORM_NONE;
  P.self_out = out;
  return launch(P, pl, c.n_levels, c.order, st);
}

}  // namespace sk
