// Untruncated signature kernel by the Goursat-PDE finite-difference solve
// (the reference's `algorithm="pde"`: _pde_stream / _pde_gram, kernels.py:334-507).
//
// On the node grid k = 0..T1, l = 0..T2 (T = L-1, or L when difference=False)
// with K(0, l) = K(k, 0) = 1, every interior node is
//   both   = K(k, l-1) + K(k-1, l)
//   K(k,l) = both - K(k-1, l-1) + 0.5 * C(k, l) * both
// with C(k, l) the double difference G(k,l) - G(k-1,l) - G(k,l-1) + G(k-1,l-1)
// of the point kernel (difference=True) or the raw point kernel
// k(x_{k-1}, y_{l-1}) (difference=False), kernels.py:369-397. The reference
// sweeps antidiagonals with three diagonals of state; here one thread owns one
// pair and sweeps rows, keeping one row of K and one row of G (O(L') state in
// the workspace, pair index fastest so warps access it coalesced). The update
// is evaluated in the reference's operation order without FMA contraction.
// Float64 throughout; this is the reference-parity path for `pde`.
#include <algorithm>

#include "sk_common.cuh"

namespace sk {
namespace {

constexpr int PDE_THREADS = 128;

struct PdeParams {
  const double *X, *Y;
  int64_t nx, lx, ny, ly, d;
  int64_t t1, t2;
  StaticF64 S;
  int difference;
  int mode;  // 0 rect pairs, 1 symmetric (j >= i), 2 paired (i == j)
  int64_t row_begin;
  int64_t g0, count;
  double *scratch;  // [slot][count]: K row (t2+1), G row (ly)
  double *out;      // [count] kernel values of this chunk
};

__global__ void __launch_bounds__(PDE_THREADS) pde_kernel(PdeParams P) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  const int64_t g = P.g0 + t;
  int64_t i, j;
  if (P.mode == 2) {
    i = j = g;
  } else {
    i = P.row_begin + g / P.ny;
    j = g % P.ny;
  }
  if (P.mode == 1 && j < i) {  // lower triangle of a symmetric Gram is mirrored
    P.out[t] = 0.0;
    return;
  }
  const int64_t CH = P.count, T1 = P.t1, T2 = P.t2;
  const double *xs = P.X + i * P.lx * P.d;
  const double *ys = (P.mode == 2 ? P.X : P.Y) + j * P.ly * P.d;
  double *Kr = P.scratch + t;            // K(k-1, l), l = 0..T2
  double *Gp = Kr + (T2 + 1) * CH;       // G(k-1, c), c = 0..ly-1 (difference only)
  for (int64_t l = 0; l <= T2; ++l) Kr[l * CH] = 1.0;
  if (P.difference)
    for (int64_t c = 0; c < P.ly; ++c) Gp[c * CH] = static_eval_f64(P.S, xs, ys + c * P.d, (int)P.d);
  for (int64_t k = 1; k <= T1; ++k) {
    double diag = Kr[0];  // K(k-1, 0)
    double left = 1.0;    // K(k, 0)
    double g_left = 0.0;  // G(k, l-1)
    const double *xk = xs + (P.difference ? k : k - 1) * P.d;
    if (P.difference) {
      g_left = static_eval_f64(P.S, xk, ys, (int)P.d);  // G(k, 0)
    }
    for (int64_t l = 1; l <= T2; ++l) {
      double C;
      if (P.difference) {
        const double g11 = static_eval_f64(P.S, xk, ys + l * P.d, (int)P.d);  // G(k, l)
        const double g01 = Gp[l * CH];                                         // G(k-1, l)
        const double g00 = Gp[(l - 1) * CH];                                   // G(k-1, l-1)
        C = __dadd_rn(__dsub_rn(__dsub_rn(g11, g01), g_left), g00);
        Gp[(l - 1) * CH] = g_left;  // row k replaces row k-1 behind the sweep
        if (l == T2) Gp[l * CH] = g11;
        g_left = g11;
      } else {
        C = static_eval_f64(P.S, xk, ys + (l - 1) * P.d, (int)P.d);
      }
      const double up = Kr[l * CH];  // K(k-1, l)
      const double both = __dadd_rn(left, up);
      const double knew = __dadd_rn(__dsub_rn(both, diag), __dmul_rn(__dmul_rn(0.5, C), both));
      diag = up;
      Kr[l * CH] = knew;
      left = knew;
    }
    if (P.difference && T2 == 0) Gp[0] = g_left;
  }
  P.out[t] = Kr[T2 * CH];
}

// out[t] -> K (cross / symmetric with mirror) or self values
__global__ void pde_scatter_kernel(PdeParams P, double *K, int64_t ldk, double *self_out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  const int64_t g = P.g0 + t;
  const double v = P.out[t];
  if (P.mode == 2) {
    self_out[g] = v;
    return;
  }
  const int64_t i = P.row_begin + g / P.ny, j = g % P.ny;
  if (P.mode == 1) {
    if (j < i) return;
    K[i * ldk + j] = v;
    K[j * ldk + i] = v;
  } else {
    K[(i - P.row_begin) * ldk + j] = v;
  }
}

// --- warp per pair, systolic over the columns (T2 <= 32 * 8) -------------
// Lane q owns the C nodes l = qC+1 .. qC+C of every row and runs row k at
// step k + q: its left neighbour finished row k (and handed over K(k, qC) and
// G(k, qC) by shuffle) one step earlier, so the whole solve is T1 + 31 steps
// with every state in registers; the point kernel is evaluated once per node
// (the column-0 values, which no lane owns, are formed up front into shared
// memory). Same float64 update, same operation order as pde_kernel.
constexpr int PDE_WARPS = 8;
constexpr int PDE_CMAX = 8;
constexpr int PDE_G0 = 32 * PDE_CMAX + 1;  // column-0 values per warp (rows 0..T1)

// DB > 0 (d <= DB, C * DB <= 32): the own nodes' y points and squared norms
// are held in registers for the whole pair and each row's x point and norm
// are loaded once per step (the evaluation is then d FMAs and the kind's
// function, bitwise the static_eval_f64 arithmetic); DB = 0 evaluates from
// memory.
template <int C, int DB>
__global__ void __launch_bounds__(32 * PDE_WARPS) pde_warp_kernel(PdeParams P, int64_t npairs,
                                                                  double *K, int64_t ldk,
                                                                  double *self_out) {
  __shared__ double g0s[PDE_WARPS][PDE_G0];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t T1 = P.t1, T2 = P.t2;
  const int d = (int)P.d;
  const bool diff = P.difference;
  const int64_t nl = (T2 + C - 1) / C;  // lanes with nodes
  const int64_t c0 = (int64_t)lane * C;
  const int n = (int)(c0 >= T2 ? 0 : (T2 - c0 < C ? T2 - c0 : C));
  for (int64_t g = (int64_t)blockIdx.x * PDE_WARPS + warp; g < npairs;
       g += (int64_t)gridDim.x * PDE_WARPS) {
    int64_t i, j;
    if (P.mode == 2) {
      i = j = g;
    } else {
      i = P.row_begin + g / P.ny;
      j = g % P.ny;
      if (P.mode == 1 && j < i) continue;  // warp-uniform
    }
    const double *xs = P.X + i * P.lx * d;
    const double *ys = (P.mode == 2 ? P.X : P.Y) + j * P.ly * d;
    double v = 1.0;
    if (T1 > 0 && T2 > 0) {
      if (diff) {  // G(k, 0), k = 0..T1
        for (int64_t k = lane; k <= T1; k += 32) g0s[warp][k] = static_eval_f64(P.S, xs + k * d, ys, d);
        __syncwarp();
      }
      constexpr int DR = DB > 0 ? DB : 1;
      const bool inner = P.S.kind == SK_LINEAR || P.S.kind == SK_POLYNOMIAL;
      double yr[C][DR], yyr[C], xr[DR], xx = 0.0;
      if constexpr (DB > 0) {
#pragma unroll
        for (int q = 0; q < C; ++q) {
          const int64_t yl = q < n ? (diff ? c0 + q + 1 : c0 + q) : 0;
          yyr[q] = 0.0;
#pragma unroll
          for (int k = 0; k < DB; ++k) {
            yr[q][k] = k < d ? ys[yl * d + k] : 0.0;
            if (k < d) yyr[q] = fma(yr[q][k], yr[q][k], yyr[q]);
          }
        }
      }
      // the point kernel of this row's x (xr, xx) and own node q
      const auto eval_own = [&](int q) -> double {
        double xy = 0.0;
#pragma unroll
        for (int k = 0; k < DR; ++k)
          if (k < d) xy = fma(xr[k], yr[q][k], xy);
        return inner ? static_from_inner(P.S, xy) : static_from_sq(P.S, xx + yyr[q] - 2.0 * xy);
      };
      double kup[C], gp[C];  // K(k-1, l), G(k-1, l) of the own nodes
#pragma unroll
      for (int q = 0; q < C; ++q) {
        kup[q] = 1.0;
        gp[q] = (diff && q < n) ? static_eval_f64(P.S, xs, ys + (c0 + q + 1) * d, d) : 0.0;
      }
      // K(k, last own node), G(k, last own node): row 0 to start with
      double myK = 1.0, myG = 0.0;
#pragma unroll
      for (int q = 0; q < C; ++q)
        if (q == n - 1) myG = gp[q];
      double inK_prev = 1.0, inG_prev = 0.0;  // the left neighbour's row k-1 hand-over
      for (int64_t s = 1; s <= T1 + nl - 1; ++s) {
        const double inK = __shfl_up_sync(0xffffffffu, myK, 1);
        const double inG = __shfl_up_sync(0xffffffffu, myG, 1);
        const int64_t k = s - lane;
        if (k >= 1 && k <= T1 && n > 0) {
          double left, diag, gl, gd;  // K(k, c0), K(k-1, c0), G(k, c0), G(k-1, c0)
          if (lane == 0) {
            left = 1.0;
            diag = 1.0;
            gl = diff ? g0s[warp][k] : 0.0;
            gd = diff ? g0s[warp][k - 1] : 0.0;
          } else {
            left = inK;
            diag = inK_prev;
            gl = inG;
            gd = inG_prev;
          }
          const double *xk = xs + (diff ? k : k - 1) * d;
          if constexpr (DB > 0) {
            xx = 0.0;
#pragma unroll
            for (int kk = 0; kk < DB; ++kk) {
              xr[kk] = kk < d ? xk[kk] : 0.0;
              if (kk < d) xx = fma(xr[kk], xr[kk], xx);
            }
          }
#pragma unroll
          for (int q = 0; q < C; ++q) {
            if (q < n) {
              const int64_t l = c0 + q + 1;
              double Cv;
              if (diff) {
                const double g11 = DB > 0 ? eval_own(q)
                                          : static_eval_f64(P.S, xk, ys + l * d, d);  // G(k, l)
                Cv = __dadd_rn(__dsub_rn(__dsub_rn(g11, gp[q]), gl), gd);
                gd = gp[q];
                gp[q] = g11;
                gl = g11;
              } else {
                Cv = DB > 0 ? eval_own(q) : static_eval_f64(P.S, xk, ys + (l - 1) * d, d);
              }
              const double up = kup[q];
              const double both = __dadd_rn(left, up);
              const double knew =
                  __dadd_rn(__dsub_rn(both, diag), __dmul_rn(__dmul_rn(0.5, Cv), both));
              diag = up;
              kup[q] = knew;
              left = knew;
            }
          }
          myK = left;
          myG = gl;
          inK_prev = inK;
          inG_prev = inG;
        } else if (k == 0) {
          inK_prev = inK;  // row 0 of the left neighbour: K = 1, G(0, c0)
          inG_prev = inG;
        }
      }
      // K(T1, T2): the lane owning node T2, after its last row
      const int owner = (int)((T2 - 1) / C);
      v = __shfl_sync(0xffffffffu, myK, owner);
    }
    if (lane == 0) {
      if (P.mode == 2) {
        self_out[g] = v;
      } else if (P.mode == 1) {
        K[i * ldk + j] = v;
        K[j * ldk + i] = v;
      } else {
        K[(i - P.row_begin) * ldk + j] = v;
      }
    }
    __syncwarp();  // g0s is rewritten by the next pair
  }
}

int run_pde_warp(PdeParams P, int64_t npairs, double *K, int64_t ldk, double *self_out,
                 cudaStream_t st) {
  const int64_t C = (P.t2 + 31) / 32;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((npairs + PDE_WARPS - 1) / PDE_WARPS,
                                                              (int64_t)sm_count() * 16));
  const int64_t cc = C <= 1 ? 1 : (C <= 2 ? 2 : (C <= 4 ? 4 : 8));
  int64_t db = P.d <= 4 ? 4 : (P.d <= 8 ? 8 : (P.d <= 16 ? 16 : 0));
  if (cc * db > 32) db = 0;  // register budget: the generic evaluation
#define SK_PW(CC, DD)                                                                         \
  if (cc == CC && db == DD)                                                                   \
    pde_warp_kernel<CC, DD><<<(unsigned)grid, 32 * PDE_WARPS, 0, st>>>(P, npairs, K, ldk, self_out);
  SK_PW(1, 4) SK_PW(1, 8) SK_PW(1, 16) SK_PW(2, 4) SK_PW(2, 8) SK_PW(2, 16) SK_PW(4, 4)
  SK_PW(4, 8) SK_PW(8, 4)
  SK_PW(1, 0) SK_PW(2, 0) SK_PW(4, 0) SK_PW(8, 0)
#undef SK_PW
  SK_CHECK_LAUNCH();
  return SK_OK;
}

int64_t pde_slots(int64_t t2, int64_t ly) { return (t2 + 1) + ly + 1; }

int64_t pde_chunk(int64_t npairs, int64_t slots) {
  const int64_t per = slots * 8;
  int64_t ch = std::max<int64_t>(1024, (256ll << 20) / per);
  ch = std::min<int64_t>(ch, 1 << 16);
  return std::max<int64_t>(1, std::min(ch, npairs));
}

int run_pde(PdeParams P, int64_t npairs, double *K, int64_t ldk, double *self_out, void *ws,
            size_t ws_bytes, cudaStream_t st) {
  if (npairs <= 0) return SK_OK;
  if (P.t2 <= 32 * PDE_CMAX && P.t1 <= 32 * PDE_CMAX) return run_pde_warp(P, npairs, K, ldk, self_out, st);
  const int64_t slots = pde_slots(P.t2, P.ly);
  const int64_t ch = pde_chunk(npairs, slots);
  const size_t need = (size_t)ch * slots * sizeof(double);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small for the pde path: need " +
                                      std::to_string(need) + " bytes");
  P.scratch = (double *)ws;
  P.out = P.scratch + ch * (slots - 1);
  for (int64_t g0 = 0; g0 < npairs; g0 += ch) {
    P.g0 = g0;
    P.count = std::min(ch, npairs - g0);
    const unsigned blocks = (unsigned)((P.count + PDE_THREADS - 1) / PDE_THREADS);
    pde_kernel<<<blocks, PDE_THREADS, 0, st>>>(P);
    SK_CHECK_LAUNCH();
    pde_scatter_kernel<<<blocks, PDE_THREADS, 0, st>>>(P, K, ldk, self_out);
    SK_CHECK_LAUNCH();
  }
  return SK_OK;
}

PdeParams pde_params(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                     int64_t ly, int64_t d, const sk_static_spec &sp, int difference) {
  PdeParams P{};
  P.X = X;
  P.Y = Y;
  P.nx = nx;
  P.lx = lx;
  P.ny = ny;
  P.ly = ly;
  P.d = d;
  P.S = to_static(sp);
  P.difference = difference;
  P.t1 = difference ? lx - 1 : lx;
  P.t2 = difference ? ly - 1 : ly;
  return P;
}

}  // namespace

size_t pde_workspace_bytes(int64_t npairs, int64_t ly, int difference) {
  const int64_t t2 = difference ? std::max<int64_t>(ly - 1, 0) : ly;
  const int64_t slots = pde_slots(t2, ly);
  return (size_t)pde_chunk(std::max<int64_t>(npairs, 1), slots) * slots * sizeof(double);
}

int pde_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
             int64_t d, int symmetric, const sk_static_spec &sp, int difference,
             int64_t row_begin, int64_t row_end, double *K, int64_t ldk, void *ws,
             size_t ws_bytes, cudaStream_t st) {
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  }
  PdeParams P = pde_params(X, nx, lx, Y, ny, ly, d, sp, difference);
  P.mode = symmetric ? 1 : 0;
  P.row_begin = row_begin;
  return run_pde(P, (row_end - row_begin) * ny, K, ldk, nullptr, ws, ws_bytes, st);
}

int pde_self(const double *X, int64_t n, int64_t l, int64_t d, const sk_static_spec &sp,
             int difference, double *out, void *ws, size_t ws_bytes, cudaStream_t st) {
  PdeParams P = pde_params(X, n, l, X, n, l, d, sp, difference);
  P.mode = 2;
  return run_pde(P, n, nullptr, 0, out, ws, ws_bytes, st);
}

}  // namespace sk
