// Host side of the fused FP32 path: shape planning, input packing and launch.
#include <algorithm>
#include <cmath>

#include "sk_fast.cuh"

namespace sk {
namespace fast {

__global__ void pack_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                            int64_t Lp, int D, int DP, double coord_scale, int with_norm,
                            float *__restrict__ out) {
  const int64_t total = n * Lp;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t / Lp;
    const int64_t pt = min(t % Lp, L - 1);  // repeat the last point (zero increments)
    const double *src = X + (s * L + pt) * d;
    float *dst = out + t * DP;
    double nrm = 0.0;
    for (int k = 0; k < D; ++k) {
      const float v = (k < d) ? (float)(src[k] * coord_scale) : 0.f;
      dst[k] = v;
      nrm += (double)v * (double)v;  // n-term from the rounded coordinates
    }
    dst[D] = with_norm ? (float)(-0.5 * nrm) : 0.f;
    for (int k = D + 1; k < DP; ++k) dst[k] = 0.f;
  }
}

namespace {

constexpr int RX_MULTI = 8;  // x sequences per tile when the carry buffer is in use

struct Plan {
  bool ok = false;
  int D = 0, DP = 0, sw = 0, segs = 0, npanel = 1, nhp = 0;
  bool linear = false;
};

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

constexpr size_t SMEM_LIMIT = 200 * 1024;

Plan plan_for(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  Plan pl;
  const int kind = c.static_spec.kind;
  if (c.precision != SK_PREC_FP32 || !c.difference) return pl;
  if (kind != SK_RBF && kind != SK_LINEAR) return pl;
  if (c.n_levels < 1 || c.n_levels > 8 || c.order != 1) return pl;
  if (d < 1 || d > 16 || lx < 2 || ly < 2) return pl;
  pl.D = d <= 4 ? 4 : (d <= 8 ? 8 : 16);
  pl.DP = pl.D + 4;
  if (ly <= 32 * C) {
    pl.sw = next_pow2((int)((ly + C - 1) / C));
  } else {  // sequential 256-column panels with chain carries through HBM/L2
    pl.sw = 32;
    pl.npanel = (int)((ly + 32 * C - 1) / (32 * C));
    const int nca = c.n_levels >= 2 ? c.n_levels - 1 : 0;
    pl.nhp = (nca + 2 + 3) / 4 * 4;
  }
  if (lx < pl.sw) return pl;
  // + one pad row: the row prefetch may read one row past the last slot
  if (((size_t)NSLOT * lx + 1) * pl.DP * sizeof(float) > SMEM_LIMIT) return pl;
  pl.segs = NWARPS * (32 / pl.sw);
  pl.linear = kind == SK_LINEAR;
  pl.ok = true;
  return pl;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int lyp_of(const Plan &pl) { return pl.sw * C * pl.npanel; }

size_t carry_bytes(int64_t lx, const Plan &pl) {
  if (pl.npanel <= 1) return 0;
  return align256((size_t)sm_count() * NWARPS * (RX_MULTI + 2) * lx * pl.nhp * sizeof(float));
}

double coord_scale(const sk_kernel_config &c) {
  if (c.static_spec.kind == SK_LINEAR) return std::sqrt(c.static_spec.scale);
  // G = exp(-|x-y|^2 / (2 bw^2)) = exp2(-|x'-y'|^2 / 2) with x' = x sqrt(log2 e) / bw
  return std::sqrt(1.4426950408889634) / c.static_spec.bandwidth;
}

int pack(const double *X, int64_t n, int64_t L, int64_t d, int64_t Lp, const Plan &pl,
         const sk_kernel_config &c, float *out, cudaStream_t st) {
  const int64_t total = n * Lp;
  if (total <= 0) return SK_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 16);
  pack_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, n, L, d, Lp, pl.D, pl.DP, coord_scale(c),
                                                 pl.linear ? 0 : 1, out);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

int launch(const Params &P, const Plan &pl, int M, cudaStream_t st) {
  // + one pad row: the row prefetch may read one row past the last slot
  const size_t smem = ((size_t)NSLOT * P.lx + 1) * pl.DP * sizeof(float);
  switch (pl.D) {
    case 4:
      return launch_d4(P, M, pl.linear, smem, st);
    case 8:
      return launch_d8(P, M, pl.linear, smem, st);
    case 16:
      return launch_d16(P, M, pl.linear, smem, st);
    default:
      return fail(SK_ERR_UNSUPPORTED, "fast path: unsupported channel padding");
  }
}

// Pack both roles into the workspace: x rows [rows][lxp], y columns [n][lyp]
// (one shared array when x and y are the same sequences).
struct Packed {
  const float *xs, *ys;
  int lxp, lyp;
  float *carry;
};

int pack_roles(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
               int64_t ly, int64_t d, bool same, const Plan &pl, const sk_kernel_config &c,
               void *ws, size_t ws_bytes, cudaStream_t st, Packed &out) {
  const int64_t lyp = lyp_of(pl);
  size_t need;
  if (same) {
    const int64_t Lp = std::max<int64_t>(lx, lyp);
    const size_t b = align256((size_t)nx * Lp * pl.DP * 4);
    need = b + carry_bytes(lx, pl);
    if (!ws || ws_bytes < need)
      return fail(SK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    int rc = pack(X, nx, lx, d, Lp, pl, c, (float *)ws, st);
    if (rc) return rc;
    out.xs = out.ys = (const float *)ws;
    out.lxp = out.lyp = (int)Lp;
    out.carry = (float *)((char *)ws + b);
  } else {
    const size_t bx = align256((size_t)nx * lx * pl.DP * 4);
    const size_t by = align256((size_t)ny * lyp * pl.DP * 4);
    need = bx + by + carry_bytes(lx, pl);
    if (!ws || ws_bytes < need)
      return fail(SK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need));
    float *xsb = (float *)ws;
    float *ysb = (float *)((char *)ws + bx);
    int rc = pack(X, nx, lx, d, lx, pl, c, xsb, st);
    if (rc) return rc;
    rc = pack(Y, ny, ly, d, lyp, pl, c, ysb, st);
    if (rc) return rc;
    out.xs = xsb;
    out.ys = ysb;
    out.lxp = (int)lx;
    out.lyp = (int)lyp;
    out.carry = (float *)((char *)ws + bx + by);
  }
  return SK_OK;
}

Params base_params(const Plan &pl, const Packed &pk, int64_t lx) {
  Params P{};
  P.xs = pk.xs;
  P.ys = pk.ys;
  P.lxp = pk.lxp;
  P.lyp = pk.lyp;
  P.lx = (int)lx;
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
  using namespace fast;
  size_t need = 0;
  const Plan px = plan_for(lx, lx, d, c);
  if (px.ok)  // self levels of X (also the symmetric Gram)
    need = std::max(need, align256((size_t)nx * std::max<int64_t>(lx, lyp_of(px)) * px.DP * 4) +
                              carry_bytes(lx, px));
  if (ny > 0) {
    const Plan py = plan_for(ly, ly, d, c);
    if (py.ok)
      need = std::max(need, align256((size_t)ny * std::max<int64_t>(ly, lyp_of(py)) * py.DP * 4) +
                                carry_bytes(ly, py));
    const Plan pg = plan_for(lx, ly, d, c);
    if (pg.ok)
      need = std::max(need, align256((size_t)nx * lx * pg.DP * 4) +
                                align256((size_t)ny * lyp_of(pg) * pg.DP * 4) + carry_bytes(lx, pg));
  }
  return need;
}

int fast_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
              int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
              int64_t row_begin, int64_t row_end, const double *diag_x, const double *diag_y,
              double *K, int64_t ldk, double *levels, void *ws, size_t ws_bytes,
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
  int rc = pack_roles(X, nx, lx, Y, ny, ly, d, symmetric != 0, pl, c, ws, ws_bytes, st, pk);
  if (rc) return rc;
  Params P = base_params(pl, pk, lx);
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
  return launch(P, pl, c.n_levels, st);
}

int fast_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                     const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                     cudaStream_t st) {
  using namespace fast;
  const Plan pl = plan_for(l, l, d, c);
  if (!pl.ok) return fail(SK_ERR_UNSUPPORTED, "fast path does not cover this configuration");
  if (n <= 0) return SK_OK;
  Packed pk{};
  int rc = pack_roles(X, n, l, X, n, l, d, true, pl, c, ws, ws_bytes, st, pk);
  if (rc) return rc;
  // each CTA evaluates its segments' y against the same sequences as x and
  // keeps the diagonal: the same kernel and arithmetic as the Gram's diagonal
  Params P = base_params(pl, pk, l);
  P.nx = P.ny = n;
  P.tiles_y = (n + pl.segs - 1) / pl.segs;
  P.ntiles = P.tiles_y;
  P.rx = pl.segs;
  P.row_begin = 0;
  P.row_end = n;
  P.diag_mode = 1;
  P.norm = SK_NORM_NONE;
  P.self_out = out;
  return launch(P, pl, c.n_levels, st);
}

}  // namespace sk
