// General float64 path: any static kind, any order p <= GEN_MAX_ORDER, any
// n_levels <= GEN_MAX_LEVELS, difference on/off, per-level increment lists.
//
// One thread owns one sequence pair and sweeps its T1 x T2 increment grid row
// by row, carrying only column accumulators (O(T2) state) instead of the
// reference's full (p, p, T1, T2) state tensors (kernels.py:175-199). The
// recursion is exactly the reference's (kernels.py:179-199):
//   R'[0,0] = A * S(C),            C = sum_{q,r} R[q,r], S = 2-D exclusive prefix
//   R'[q,0] = A/(q+1) * E_j(sum_r R[q-1,r])
//   R'[0,q] = A/(q+1) * E_i(sum_q' R[q',q-1])
//   R'[q,r] = A/((q+1)(r+1)) * R[q-1,r-1]
// evaluated cell by cell: S(C)(i,j) is a running row sum of the column
// accumulators colC(j) = sum_{i'<i} C(i',j); E_j is a running row sum; E_i is
// a column accumulator. Per-thread column state lives in the workspace with
// the pair index fastest, so a warp's accesses are coalesced.
//
// This path is the float64 (bit-level) reference-parity path and the
// fallback for configurations the fused FP32 kernels do not instantiate.

#include <algorithm>
#include <cstdio>

#include "sk_common.cuh"

namespace sk {

namespace {

constexpr int GEN_THREADS = 128;

struct GenParams {
  // point inputs (mode 0..2) or increment input (mode 3)
  const double *X;
  const double *Y;
  const double *A;
  int64_t nx, lx, ny, ly, d;
  int64_t t1, t2;  // increment grid
  StaticF64 S;
  int M, p, difference, per_level;
  int mode;  // 0 rect pairs, 1 symmetric (j >= i), 2 paired (i == j), 3 increments
  // lifted (rfsf_exact_gram, features.py:397-424): X/Y hold per-slot static
  // features concatenated along the channel axis; level m's point kernel is the
  // inner product of slot m's features, channels [woff[m-1], woff[m]).
  int lifted;
  int woff[GEN_MAX_LEVELS + 1];
  // lifted with precomputed slot Grams (lifted_gram): G[h][(i - g_row0) * lx + r][j * ly + c]
  // = <phi_h(x_i[r]), phi_h(y_j[c])>, written by dgemm_nt_kernel
  const double *G;
  int64_t g_ld, g_lvl, g_row0;
  int64_t row_begin;
  int64_t g0, count;  // pair ids [g0, g0+count) of this chunk
  double *scratch;    // [slot][count]
  double *lv;         // [count][M+1]
};

__device__ inline void pair_of(const GenParams &P, int64_t g, int64_t &i, int64_t &j) {
  if (P.mode == 2 || P.mode == 3) {
    i = g;
    j = g;
  } else {
    i = P.row_begin + g / P.ny;
    j = g % P.ny;
  }
}

// inner product of slot h's features of two points (level h+1's lifted point kernel)
__device__ inline double lifted_dot(const GenParams &P, int h, const double *x, const double *y) {
  double acc = 0.0;
  for (int k = P.woff[h]; k < P.woff[h + 1]; ++k) acc = fma(x[k], y[k], acc);
  return acc;
}

// Level values of pair (i, j) (pair id g) into out[0..M]; this thread's
// column state is scratch slot t of CH interleaved slots.
__device__ void pair_levels(const GenParams &P, int64_t g, int64_t i, int64_t j, int64_t t,
                            int64_t CH, double *out) {
  const int M = P.M;
  out[0] = 1.0;
  for (int m = 1; m <= M; ++m) out[m] = 0.0;
  const int64_t T1 = P.t1, T2 = P.t2;
  if (M == 0 || T1 <= 0 || T2 <= 0) return;
  const int p = P.p;

  // workspace slots: colC[(m-1)*T2 + j] m=1..M-1, colSY[((m-1)*(p-1)+r)*T2 + j], Gprev[ly]
  double *colC = P.scratch + t;
  double *colSY = colC + (int64_t)(M - 1) * T2 * CH;
  double *Gprev = colSY + (int64_t)(M - 1) * (p - 1) * T2 * CH;
  for (int64_t k = 0; k < (int64_t)(M - 1) * T2 * p; ++k) colC[k * CH] = 0.0;
  const bool lifted = P.lifted != 0;
  const bool gmode = lifted && P.G != nullptr;  // slot Grams precomputed
  const int nG = lifted ? M : 1;  // Gprev rows (one per level when lifted)
  const double *gx = !gmode        ? nullptr
                     : P.mode == 2 ? P.G + i * P.lx * P.g_ld  // per-sequence self Grams
                                   : P.G + ((i - P.g_row0) * P.lx) * P.g_ld + j * P.ly;

  const double *xs = nullptr, *ys = nullptr;
  const bool from_points = P.mode != 3;
  if (from_points) {
    xs = P.X + i * P.lx * P.d;
    ys = (P.mode == 2 ? P.X : P.Y) + j * P.ly * P.d;
    if (P.difference && !gmode)
      for (int h = 0; h < nG; ++h)
        for (int64_t c = 0; c < P.ly; ++c)
          Gprev[(h * P.ly + c) * CH] = lifted ? lifted_dot(P, h, xs, ys + c * P.d)
                                              : static_eval_f64(P.S, xs, ys + c * P.d, (int)P.d);
  }
  double gl_lev[GEN_MAX_LEVELS], a_lev[GEN_MAX_LEVELS];

  double s2d[GEN_MAX_LEVELS];
  double ex[GEN_MAX_LEVELS * GEN_MAX_ORDER];
  double Ra[GEN_MAX_ORDER * GEN_MAX_ORDER], Rb[GEN_MAX_ORDER * GEN_MAX_ORDER];
  double lsum[GEN_MAX_LEVELS + 1];
  for (int m = 0; m <= M; ++m) lsum[m] = 0.0;

  for (int64_t r = 0; r < T1; ++r) {
    for (int m = 0; m < M; ++m) s2d[m] = 0.0;
    for (int k = 0; k < M * p; ++k) ex[k] = 0.0;
    const double *xa = nullptr;
    double gl = 0.0;  // G(r+1, c) of the previous column
    if (from_points && P.difference && !gmode) {
      xa = xs + (r + 1) * P.d;
      if (lifted)
        for (int h = 0; h < M; ++h) gl_lev[h] = lifted_dot(P, h, xa, ys);
      else
        gl = static_eval_f64(P.S, xa, ys, (int)P.d);
    }
    for (int64_t c = 0; c < T2; ++c) {
      double a_shared = 0.0;
      if (gmode) {
        // per-level double difference of the slot Grams (features.py:418-419)
        for (int h = 0; h < M; ++h) {
          const double *gh = gx + h * P.g_lvl;
          if (P.difference) {
            const double g11 = gh[(r + 1) * P.g_ld + c + 1], g01 = gh[r * P.g_ld + c + 1];
            const double g10 = gh[(r + 1) * P.g_ld + c], g00 = gh[r * P.g_ld + c];
            a_lev[h] = g11 - g01 - g10 + g00;
          } else {
            a_lev[h] = gh[r * P.g_ld + c];
          }
        }
      } else if (lifted) {
        // per-level double difference of the slot inner products (features.py:418-419)
        for (int h = 0; h < M; ++h) {
          if (P.difference) {
            double *gp = Gprev + (int64_t)h * P.ly * CH;
            const double g11 = lifted_dot(P, h, xa, ys + (c + 1) * P.d);
            const double g01 = gp[(c + 1) * CH];
            const double g00 = gp[c * CH];
            a_lev[h] = g11 - g01 - gl_lev[h] + g00;
            gp[c * CH] = gl_lev[h];
            if (c == T2 - 1) gp[(c + 1) * CH] = g11;
            gl_lev[h] = g11;
          } else {
            a_lev[h] = lifted_dot(P, h, xs + r * P.d, ys + c * P.d);
          }
        }
      } else if (from_points) {
        if (P.difference) {
          // kernels.py:281: G[1:,1:] - G[:-1,1:] - G[1:,:-1] + G[:-1,:-1]
          const double g11 = static_eval_f64(P.S, xa, ys + (c + 1) * P.d, (int)P.d);
          const double g01 = Gprev[(c + 1) * CH];
          const double g00 = Gprev[c * CH];
          a_shared = g11 - g01 - gl + g00;
          Gprev[c * CH] = gl;
          if (c == T2 - 1) Gprev[(c + 1) * CH] = g11;
          gl = g11;
        } else {
          a_shared = static_eval_f64(P.S, xs + r * P.d, ys + c * P.d, (int)P.d);
        }
      } else if (!P.per_level) {
        a_shared = P.A[(g * T1 + r) * T2 + c];
      }
      double *Rp = Ra, *Rc = Rb;  // Rp: level m-1 at this cell, Rc: level m
      for (int m = 1; m <= M; ++m) {
        const double am =
            lifted ? a_lev[m - 1]
            : (from_points || !P.per_level)
                ? a_shared
                : P.A[(((int64_t)(m - 1) * P.count + g) * T1 + r) * T2 + c];
        for (int k = 0; k < p * p; ++k) Rc[k] = 0.0;
        if (m == 1) {
          Rc[0] = am;
        } else {
          const int mm = m - 2;  // index of level m-1 in the accumulators
          double Ctot = 0.0;
          for (int k = 0; k < p * p; ++k) Ctot += Rp[k];
          double *cc = colC + ((int64_t)mm * T2 + c) * CH;
          const double old = *cc;
          const double S2 = s2d[mm];
          s2d[mm] += old;
          *cc = old + Ctot;
          Rc[0] = am * S2;
          for (int q = 1; q < p; ++q) {
            double sx = 0.0, sy = 0.0;
            for (int r2 = 0; r2 < p; ++r2) sx += Rp[(q - 1) * p + r2];
            for (int q2 = 0; q2 < p; ++q2) sy += Rp[q2 * p + (q - 1)];
            double &e = ex[mm * p + (q - 1)];
            const double E = e;
            e += sx;
            double *cy = colSY + (((int64_t)mm * (p - 1) + (q - 1)) * T2 + c) * CH;
            const double oldy = *cy;
            *cy = oldy + sy;
            Rc[q * p] = (am / (q + 1)) * E;
            Rc[q] = (am / (q + 1)) * oldy;
          }
          for (int q = 1; q < p; ++q)
            for (int r2 = 1; r2 < p; ++r2)
              Rc[q * p + r2] = (am / ((q + 1) * (r2 + 1))) * Rp[(q - 1) * p + (r2 - 1)];
        }
        double cs = 0.0;
        for (int k = 0; k < p * p; ++k) cs += Rc[k];
        lsum[m] += cs;
        double *tmp = Rp;
        Rp = Rc;
        Rc = tmp;
      }
    }
  }
  for (int m = 1; m <= M; ++m) out[m] = lsum[m];
}

__global__ void __launch_bounds__(GEN_THREADS) generic_levels_kernel(GenParams P) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  const int64_t g = P.g0 + t;
  int64_t i, j;
  pair_of(P, g, i, j);
  double *out = P.lv + t * (P.M + 1);
  if (P.mode == 1 && j < i) {  // lower triangle of a symmetric Gram is mirrored
    out[0] = 1.0;
    for (int m = 1; m <= P.M; ++m) out[m] = 0.0;
    return;
  }
  pair_levels(P, g, i, j, t, P.count, out);
}

// FP32 certification pass (sk_common.cuh, fp64_fixup), after the FP32 Gram
// kernel in the same stream, one grid-stride scan over the row range of K:
//  * an entry the FP32 epilogue marked NaN (non-finite, or small against its
//    scale) is recomputed in float64 — the pair's levels and, when
//    normalised, both self levels — and written with its mirror (K(X)) and
//    its per-level output (if requested);
//  * otherwise (difference=True) the pair's exact level 1 (exact_level1, the
//    telescoped increments) is compared with the FP32 one the epilogue left
//    in k1buf: a deviation above CERT_NOISE of the entry's scale marks the
//    pair's arithmetic as noisy (float64 recompute as above), else the entry
//    is corrected to the exact level 1.
// One scratch slot per thread: no list, no host synchronisation.
struct FixupArgs {
  GenParams pair;   // mode 0 / 1 geometry of the Gram (X rows, Y columns)
  GenParams selfx;  // paired geometry over X (self levels of row sequences)
  GenParams selfy;  // ... over Y
  int norm;
  double *K;
  int64_t ldk;
  double *levels;
  int64_t rows;     // rows of the range
  const float *k1buf;  // per entry [row][ny] float2 (FP32 level 1, sum_m |k_m|), or null
  const double *diag_x, *diag_y;
};

__device__ inline void put_entry(const FixupArgs &A, int64_t row, int64_t i, int64_t j, bool sym,
                                 double v) {
  A.K[row * A.ldk + j] = v;
  if (sym && j != i) A.K[j * A.ldk + i] = v;
}

__global__ void __launch_bounds__(GEN_THREADS) fixup_kernel(FixupArgs A) {
  const GenParams &P = A.pair;
  const int M = P.M;
  const bool sym = P.mode == 1;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = A.rows * P.ny;
  double lv[GEN_MAX_LEVELS + 1], dx[GEN_MAX_LEVELS + 1], dy[GEN_MAX_LEVELS + 1];
  for (int64_t e = t; e < total; e += nthr) {
    const int64_t r = e / P.ny, j = e % P.ny;
    const int64_t i = P.row_begin + r;
    const int64_t row = sym ? i : r;
    if (sym && j < i) continue;
    double v = A.K[row * A.ldk + j];
    bool redo = isnan(v) || isinf(v);
    if (!redo && A.k1buf && !(sym && i == j)) {  // cancellation rule (write_pair's data)
      const double lim =
          A.norm == SK_NORM_NONE
              ? (double)A.k1buf[2 * (row * P.ny + j) + 1] *
                    (P.S.kind == SK_LINEAR ? CERT_TAU_RAW_LINEAR : CERT_TAU_RAW)
              : CERT_TAU_NORM;
      redo = !(fabs(v) >= lim);
    }
    if (!redo && A.k1buf && P.difference && M >= 1 && !(sym && i == j)) {
      const double k1e = exact_level1(P.S, P.X + i * P.lx * P.d, P.lx, P.Y + j * P.ly * P.d, P.ly,
                                      (int)P.d);
      const double delta = k1e - (double)A.k1buf[2 * (row * P.ny + j)];
      double scale = CERT_NOISE_RAW / CERT_NOISE * fabs(v), corr = delta;
      if (A.norm != SK_NORM_NONE) {
        const double *px = A.diag_x + i * (M + 1), *py = A.diag_y + j * (M + 1);
        scale = sqrt(fabs(px[1] * py[1]));
        if (A.norm == SK_NORM_LEVELWISE) {
          const double den = sqrt((px[1] > 0.0 ? px[1] : 0.0) * (py[1] > 0.0 ? py[1] : 0.0));
          corr = den > 0.0 ? delta / den / (double)(M + 1) : 0.0;
        } else {
          double sx = 0.0, sy = 0.0;
          for (int m = 0; m <= M; ++m) {
            sx += px[m];
            sy += py[m];
          }
          corr = delta / sqrt(sx * sy);
        }
      }
      if (fabs(delta) > CERT_NOISE * scale) {
        redo = true;
      } else {
        put_entry(A, row, i, j, sym, v + corr);
        if (A.levels) {
          A.levels[(row * A.ldk + j) * (M + 1) + 1] = k1e;
          if (sym && j != i) A.levels[(j * A.ldk + i) * (M + 1) + 1] = k1e;
        }
      }
    }
    if (!redo) continue;
    pair_levels(P, 0, i, j, t, nthr, lv);
    const double *px = nullptr, *py = nullptr;
    if (A.norm != SK_NORM_NONE) {
      pair_levels(A.selfx, 0, i, i, t, nthr, dx);
      pair_levels(A.selfy, 0, j, j, t, nthr, dy);
      px = dx;
      py = dy;
    }
    put_entry(A, row, i, j, sym, finish_entry(lv, M, A.norm, px, py));
    if (A.levels) {
      for (int m = 0; m <= M; ++m) A.levels[(row * A.ldk + j) * (M + 1) + m] = lv[m];
      if (sym && j != i)
        for (int m = 0; m <= M; ++m) A.levels[(j * A.ldk + i) * (M + 1) + m] = lv[m];
    }
  }
}

// Normalisation / level-sum epilogue for a chunk of pairs (kernels.py:586-600).
__global__ void generic_finish_kernel(GenParams P, int norm, const double *diag_x,
                                      const double *diag_y, double *K, int64_t ldk,
                                      double *levels) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.count) return;
  int64_t i, j;
  pair_of(P, P.g0 + t, i, j);
  if (P.mode == 1 && j < i) return;
  const int M = P.M;
  const double *lv = P.lv + t * (M + 1);
  const bool sym = P.mode == 1;
  const int64_t row = sym ? i : i - P.row_begin;
  if (levels) {
    for (int m = 0; m <= M; ++m) levels[(row * ldk + j) * (M + 1) + m] = lv[m];
    if (sym && j != i)
      for (int m = 0; m <= M; ++m) levels[(j * ldk + i) * (M + 1) + m] = lv[m];
  }
  if (K) {
    const double v = finish_entry(lv, M, norm, diag_x ? diag_x + i * (M + 1) : nullptr,
                                  diag_y ? diag_y + j * (M + 1) : nullptr);
    K[row * ldk + j] = v;
    if (sym && j != i) K[j * ldk + i] = v;
  }
}

__global__ void copy_levels_kernel(const double *lv, int64_t count, int M, double *out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < count * (M + 1)) out[t] = lv[t];
}

// Lifted DP with precomputed slot Grams, order 1, T' <= 128 (rfsf_exact_gram):
// one warp per pair, lanes own 4 columns, one warp-level exclusive scan per
// level and row (the order-1 recursion of pair_levels with a per-level A,
// features.py:418-424). Every level's slot-Gram row r+1 is read once (the
// previous row stays in registers) and the next row is requested before the
// current one is used; the per-pair state lives in registers instead of the
// pair-fastest workspace of the thread-per-pair kernel.
constexpr int LW_WARPS = 8;

template <int MB>
__global__ void __launch_bounds__(32 * LW_WARPS) lifted_warp_kernel(GenParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = P.M;
  const int64_t T1 = P.t1, T2 = P.t2;
  const bool diff = P.difference;
  const int c0 = 4 * lane;
  constexpr int VB = MB - 1;
  for (int64_t t = (int64_t)blockIdx.x * LW_WARPS + warp; t < P.count;
       t += (int64_t)gridDim.x * LW_WARPS) {
    const int64_t g = P.g0 + t;
    int64_t i, j;
    pair_of(P, g, i, j);
    double *out = P.lv + t * (M + 1);
    if ((P.mode == 1 && j < i) || M == 0 || T1 <= 0 || T2 <= 0) {
      if (lane == 0) {
        out[0] = 1.0;
        for (int m = 1; m <= M; ++m) out[m] = 0.0;
      }
      continue;
    }
    const double *gx = P.mode == 2 ? P.G + i * P.lx * P.g_ld
                                   : P.G + ((i - P.g_row0) * P.lx) * P.g_ld + j * P.ly;
    // G columns c0 .. c0 + 4 of one row of every level (column c0 + 4 for the
    // double difference of the lane's last cell)
    const int64_t ncol = diff ? T2 + 1 : T2;
    double gcur[MB][5], gnx[MB][5];
    const auto load_row = [&](int64_t r, double (&dst)[MB][5]) {
#pragma unroll
      for (int h = 0; h < MB; ++h)
#pragma unroll
        for (int k = 0; k < 5; ++k)
          dst[h][k] = (h < M && r < (diff ? T1 + 1 : T1) && c0 + k < ncol)
                          ? gx[h * P.g_lvl + r * P.g_ld + c0 + k]
                          : 0.0;
    };
    load_row(0, gcur);
    if (diff) load_row(1, gnx);
    double ca[VB > 0 ? VB : 1][4], lsum[MB];
#pragma unroll
    for (int m = 0; m < VB; ++m)
#pragma unroll
      for (int k = 0; k < 4; ++k) ca[m][k] = 0.0;
#pragma unroll
    for (int m = 0; m < MB; ++m) lsum[m] = 0.0;
    for (int64_t r = 0; r < T1; ++r) {
      double a[MB][4];
#pragma unroll
      for (int h = 0; h < MB; ++h)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool in = c0 + k < T2;
          // features.py:418-419: G[1:,1:] - G[:-1,1:] - G[1:,:-1] + G[:-1,:-1]
          a[h][k] = !in ? 0.0
                    : diff ? gnx[h][k + 1] - gcur[h][k + 1] - gnx[h][k] + gcur[h][k]
                           : gcur[h][k];
        }
      // advance the row window and request the next row before the recursion
      if (diff) {
#pragma unroll
        for (int h = 0; h < MB; ++h)
#pragma unroll
          for (int k = 0; k < 5; ++k) gcur[h][k] = gnx[h][k];
        load_row(r + 2, gnx);
      } else {
        load_row(r + 1, gcur);
      }
      double pre[VB > 0 ? VB : 1];
#pragma unroll
      for (int m = 0; m < VB; ++m) pre[m] = ca[m][0] + ca[m][1] + ca[m][2] + ca[m][3];
#pragma unroll
      for (int m = 0; m < VB; ++m) {
        if (m + 1 < M) {
          double inc = pre[m];
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
          }
          pre[m] = inc - pre[m];
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double Rprev = a[0][k];
        lsum[0] += Rprev;
#pragma unroll
        for (int m = 1; m < MB; ++m) {
          if (m < M) {
            const double Rn = a[m][k] * pre[m - 1];
            lsum[m] += Rn;
            pre[m - 1] += ca[m - 1][k];
            ca[m - 1][k] += Rprev;
            Rprev = Rn;
          }
        }
      }
    }
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      double v = lsum[m];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      lsum[m] = v;
    }
    if (lane == 0) {
      out[0] = 1.0;
#pragma unroll
      for (int m = 0; m < MB; ++m)
        if (m < M) out[m + 1] = lsum[m];
    }
  }
}

int64_t scratch_slots(int64_t t2, int64_t ly, int M, int p, int lifted = 0) {
  const int64_t mm = std::max(M - 1, 0);
  return mm * t2 * p + (lifted ? std::max(M, 1) : 1) * ly + 1;
}

int64_t chunk_pairs(int64_t npairs, int64_t slots, int M) {
  const int64_t per = (slots + M + 1) * 8;
  const int64_t budget = 256ll << 20;
  int64_t ch = std::max<int64_t>(1024, budget / per);
  ch = std::min<int64_t>(ch, 1 << 16);
  return std::max<int64_t>(1, std::min(ch, npairs));
}

int run_chunks(GenParams P, int64_t npairs, int norm, const double *diag_x,
               const double *diag_y, double *K, int64_t ldk, double *levels, double *self_out,
               void *ws, size_t ws_bytes, cudaStream_t st) {
  const int64_t slots = scratch_slots(P.t2, P.ly, P.M, P.p, P.lifted);
  const int64_t ch = chunk_pairs(npairs, slots, P.M);
  const size_t need = (size_t)ch * (slots + P.M + 1) * sizeof(double);
  if (ws_bytes < need || ws == nullptr)
    return fail(SK_ERR_WORKSPACE, "workspace too small for the float64 path: need " +
                                      std::to_string(need) + " bytes");
  P.scratch = (double *)ws;
  P.lv = P.scratch + ch * slots;
  for (int64_t g0 = 0; g0 < npairs; g0 += ch) {
    P.g0 = g0;
    P.count = std::min(ch, npairs - g0);
    const int blocks = (int)((P.count + GEN_THREADS - 1) / GEN_THREADS);
    if (P.lifted && P.G && P.p == 1 && P.M >= 1 && P.M <= 4 && P.t2 <= 128) {
      // (n_levels 5-8 would need 8 levels of row windows: 1.6 KB of spills)
      const unsigned wb = (unsigned)std::min<int64_t>((P.count + LW_WARPS - 1) / LW_WARPS,
                                                      (int64_t)sm_count() * 16);
      lifted_warp_kernel<4><<<wb, 32 * LW_WARPS, 0, st>>>(P);
    } else {
      generic_levels_kernel<<<blocks, GEN_THREADS, 0, st>>>(P);
    }
    SK_CHECK_LAUNCH();
    if (self_out) {
      const int64_t n = P.count * (P.M + 1);
      copy_levels_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
          P.lv, P.count, P.M, self_out + g0 * (P.M + 1));
    } else {
      generic_finish_kernel<<<blocks, GEN_THREADS, 0, st>>>(P, norm, diag_x, diag_y, K, ldk,
                                                           levels);
    }
    SK_CHECK_LAUNCH();
  }
  return SK_OK;
}

GenParams base_params(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                      int64_t ly, int64_t d, const sk_kernel_config &c) {
  GenParams P{};
  P.X = X;
  P.Y = Y;
  P.nx = nx;
  P.lx = lx;
  P.ny = ny;
  P.ly = ly;
  P.d = d;
  P.S = to_static(c.static_spec);
  P.M = c.n_levels;
  P.p = std::max(1, std::min(c.order, std::max(c.n_levels, 1)));
  P.difference = c.difference;
  P.t1 = c.difference ? std::max<int64_t>(lx - 1, 0) : lx;
  P.t2 = c.difference ? std::max<int64_t>(ly - 1, 0) : ly;
  return P;
}

}  // namespace

size_t generic_workspace_bytes(int64_t npairs, int64_t lx, int64_t ly, const sk_kernel_config &c) {
  const int M = c.n_levels;
  const int p = std::max(1, std::min(c.order, std::max(M, 1)));
  const int64_t t2 = c.difference ? std::max<int64_t>(ly - 1, 0) : ly;
  const int64_t slots = scratch_slots(t2, ly, M, p);
  const int64_t ch = chunk_pairs(std::max<int64_t>(npairs, 1), slots, M);
  (void)lx;
  return (size_t)ch * (slots + M + 1) * sizeof(double);
}

int generic_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                 int64_t ly, int64_t d, int symmetric, const sk_kernel_config &c,
                 int64_t row_begin, int64_t row_end, const double *diag_x,
                 const double *diag_y, double *K, int64_t ldk, double *levels, void *ws,
                 size_t ws_bytes, cudaStream_t st) {
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  }
  GenParams P = base_params(X, nx, lx, Y, ny, ly, d, c);
  P.mode = symmetric ? 1 : 0;
  P.row_begin = row_begin;
  const int64_t npairs = (row_end - row_begin) * ny;
  if (npairs <= 0) return SK_OK;
  return run_chunks(P, npairs, c.normalization, diag_x, diag_y, K, ldk, levels, nullptr, ws,
                    ws_bytes, st);
}

int generic_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                        const sk_kernel_config &c, double *out, void *ws, size_t ws_bytes,
                        cudaStream_t st) {
  GenParams P = base_params(X, n, l, X, n, l, d, c);
  P.mode = 2;
  if (n <= 0) return SK_OK;
  return run_chunks(P, n, SK_NORM_NONE, nullptr, nullptr, nullptr, 0, nullptr, out, ws,
                    ws_bytes, st);
}

namespace {
// Self-level fix-up: sequences whose level 0 the FP32 self-level epilogue
// marked NaN are recomputed in float64 (one thread per flagged sequence of a
// grid-stride scan).
// Self levels of the FP32 paths: level 1 -> its exact telescoped value;
// a sequence whose FP32 level 1 deviates from it by more than CERT_NOISE
// relative, or with a negative or non-finite level (self levels are >= 0),
// is recomputed in float64.
__global__ void __launch_bounds__(GEN_THREADS) self_fixup_kernel(GenParams P, int64_t n,
                                                                 double *out) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int M = P.M;
  double lv[GEN_MAX_LEVELS + 1];
  for (int64_t i = t; i < n; i += nthr) {
    double *o = out + i * (M + 1);
    bool redo = false;
    for (int m = 1; m <= M; ++m) redo |= !(o[m] >= 0.0) || isinf(o[m]);
    if (!redo && P.difference && M >= 1) {
      const double *x = P.X + i * P.lx * P.d;
      const double k1e = exact_level1(P.S, x, P.lx, x, P.lx, (int)P.d);
      if (fabs(o[1] - k1e) > CERT_NOISE * fabs(k1e))
        redo = true;
      else
        o[1] = k1e;
    }
    if (!redo) continue;
    pair_levels(P, 0, i, i, t, nthr, lv);
    for (int m = 0; m <= M; ++m) o[m] = lv[m];
  }
}
}  // namespace

namespace {
constexpr int64_t FIXUP_THREADS_MAX = 148 * 2 * GEN_THREADS;
constexpr int64_t FIXUP_SCRATCH_BUDGET = 96ll << 20;

int64_t fixup_threads(int64_t lx, int64_t ly, const sk_kernel_config &c) {
  const int M = c.n_levels;
  const int p = std::max(1, std::min(c.order, std::max(M, 1)));
  const int64_t L = std::max(lx, ly);
  const int64_t t = c.difference ? std::max<int64_t>(L - 1, 0) : L;
  const int64_t per = scratch_slots(t, L, M, p) * 8;
  const int64_t n = std::min<int64_t>(FIXUP_THREADS_MAX, FIXUP_SCRATCH_BUDGET / per);
  return std::max<int64_t>(GEN_THREADS, n / GEN_THREADS * GEN_THREADS);
}
}  // namespace

size_t fixup_workspace_bytes(int64_t lx, int64_t ly, const sk_kernel_config &c) {
  const int M = c.n_levels;
  const int p = std::max(1, std::min(c.order, std::max(M, 1)));
  const int64_t L = std::max(lx, ly);
  const int64_t t = c.difference ? std::max<int64_t>(L - 1, 0) : L;
  return (size_t)fixup_threads(lx, ly, c) * scratch_slots(t, L, M, p) * 8;
}

int fp64_fixup(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
               int64_t d, int symmetric, const sk_kernel_config &c, int64_t row_begin,
               int64_t row_end, const double *diag_x, const double *diag_y, const float *k1buf,
               double *K, int64_t ldk, double *levels, void *ws, size_t ws_bytes,
               cudaStream_t st) {
  if (!K || row_end <= row_begin || ny <= 0 || nx <= 0) return SK_OK;
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  }
  if (c.n_levels > GEN_MAX_LEVELS || c.order > GEN_MAX_ORDER)
    return fail(SK_ERR_UNSUPPORTED, "fix-up: n_levels/order beyond the float64 kernel");
  const size_t need = fixup_workspace_bytes(lx, ly, c);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small for the fix-up: need " + std::to_string(need));
  FixupArgs A{};
  A.pair = base_params(X, nx, lx, Y, ny, ly, d, c);
  A.pair.mode = symmetric ? 1 : 0;
  A.pair.row_begin = row_begin;
  A.pair.scratch = (double *)ws;
  A.selfx = base_params(X, nx, lx, X, nx, lx, d, c);
  A.selfx.mode = 2;
  A.selfx.scratch = (double *)ws;
  A.selfy = base_params(Y, ny, ly, Y, ny, ly, d, c);
  A.selfy.mode = 2;
  A.selfy.scratch = (double *)ws;
  A.norm = c.normalization;
  A.K = K;
  A.ldk = ldk;
  A.levels = levels;
  A.rows = row_end - row_begin;
  A.k1buf = k1buf;
  A.diag_x = diag_x;
  A.diag_y = symmetric ? diag_x : diag_y;
  const int64_t nthr = fixup_threads(lx, ly, c);
  fixup_kernel<<<(unsigned)(nthr / GEN_THREADS), GEN_THREADS, 0, st>>>(A);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

int fp64_self_fixup(const double *X, int64_t n, int64_t l, int64_t d, const sk_kernel_config &c,
                    double *out, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (n <= 0 || !out) return SK_OK;
  if (c.n_levels > GEN_MAX_LEVELS || c.order > GEN_MAX_ORDER)
    return fail(SK_ERR_UNSUPPORTED, "fix-up: n_levels/order beyond the float64 kernel");
  const size_t need = fixup_workspace_bytes(l, l, c);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small for the fix-up: need " + std::to_string(need));
  GenParams P = base_params(X, n, l, X, n, l, d, c);
  P.mode = 2;
  P.scratch = (double *)ws;
  const int64_t nthr = std::min<int64_t>(fixup_threads(l, l, c), (n + GEN_THREADS - 1) / GEN_THREADS * GEN_THREADS);
  self_fixup_kernel<<<(unsigned)(nthr / GEN_THREADS), GEN_THREADS, 0, st>>>(P, n, out);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

// --- rfsf_exact_gram's lifted level Grams (features.py:397-443), float64 ---------
namespace {
// C[m][n] = sum_k A[m * lda + k] * B[n * ldb + k] (float64, the slot Gram
// Ux Uy^T of _lifted_level_grams, features.py:414-415): 64 x 64 tiles, 16-wide
// K slices staged in shared memory, 4 x 4 outputs per thread.
constexpr int DG_T = 64, DG_K = 16;
__global__ void __launch_bounds__(256) dgemm_nt_kernel(const double *__restrict__ A, int64_t lda,
                                                       const double *__restrict__ B, int64_t ldb,
                                                       int64_t Mr, int64_t Nr, int K,
                                                       double *__restrict__ C, int64_t ldc,
                                                       int64_t sa = 0, int64_t sb = 0,
                                                       int64_t sc = 0) {
  __shared__ double As[DG_K][DG_T + 1], Bs[DG_K][DG_T + 1];
  A += blockIdx.z * sa;  // batch entry (per-sequence self Grams)
  B += blockIdx.z * sb;
  C += blockIdx.z * sc;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * DG_T, n0 = (int64_t)blockIdx.x * DG_T;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += DG_K) {
    for (int e = threadIdx.x; e < DG_T * DG_K; e += 256) {
      const int row = e / DG_K, kk = e % DG_K;
      const int64_t am = m0 + row, bn = n0 + row;
      const bool kin = k0 + kk < K;
      As[kk][row] = (am < Mr && kin) ? A[am * lda + k0 + kk] : 0.0;
      Bs[kk][row] = (bn < Nr && kin) ? B[bn * ldb + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < DG_K; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = As[kk][ty + 16 * u];
        b[u] = Bs[kk][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t m = m0 + ty + 16 * u, n = n0 + tx + 16 * v;
      if (m < Mr && n < Nr) C[m * ldc + n] = acc[u][v];
    }
}

constexpr size_t G_BLOCK_BYTES = (size_t)4 << 30;  // slot-Gram block budget

int64_t g_block_rows(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int M) {
  const size_t per_x = (size_t)std::max(M, 1) * lx * ny * ly * sizeof(double);
  return std::max<int64_t>(1, std::min<int64_t>(nx, (int64_t)(G_BLOCK_BYTES / std::max<size_t>(per_x, 1))));
}

int lifted_params(GenParams &P, const int64_t *slot_offsets, int M, int order) {
  if (M > GEN_MAX_LEVELS)
    return fail(SK_ERR_UNSUPPORTED, "n_levels > " + std::to_string(GEN_MAX_LEVELS));
  P.lifted = 1;
  P.S = StaticF64{};
  P.M = M;
  P.p = std::max(1, std::min(order, std::max(M, 1)));
  if (P.p > GEN_MAX_ORDER) return fail(SK_ERR_UNSUPPORTED, "order too large");
  for (int m = 0; m <= M; ++m) {
    if (slot_offsets[m] < 0 || slot_offsets[m] > P.d || (m && slot_offsets[m] < slot_offsets[m - 1]))
      return fail(SK_ERR_INVALID, "slot_offsets must be non-decreasing within [0, width]");
    P.woff[m] = (int)slot_offsets[m];
  }
  return SK_OK;
}

GenParams lifted_base(const double *UX, int64_t nx, int64_t lx, const double *UY, int64_t ny,
                      int64_t ly, int64_t width, int difference) {
  GenParams P{};
  P.X = UX;
  P.Y = UY;
  P.nx = nx;
  P.lx = lx;
  P.ny = ny;
  P.ly = ly;
  P.d = width;
  P.difference = difference;
  P.t1 = difference ? std::max<int64_t>(lx - 1, 0) : lx;
  P.t2 = difference ? std::max<int64_t>(ly - 1, 0) : ly;
  return P;
}
}  // namespace

size_t lifted_workspace_bytes(int64_t npairs, int64_t ly, int M, int order, int difference) {
  const int p = std::max(1, std::min(order, std::max(M, 1)));
  const int64_t t2 = difference ? std::max<int64_t>(ly - 1, 0) : ly;
  const int64_t slots = scratch_slots(t2, ly, M, p, 1);
  const int64_t ch = chunk_pairs(std::max<int64_t>(npairs, 1), slots, M);
  return (size_t)ch * (slots + M + 1) * sizeof(double);
}

size_t lifted_gram_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int M,
                                   int order, int difference) {
  const int64_t bx = g_block_rows(nx, lx, ny, ly, M);
  const size_t g = (size_t)std::max(M, 1) * bx * lx * ny * ly * sizeof(double);
  return lifted_workspace_bytes(bx * ny, ly, M, order, difference) + ((g + 255) & ~(size_t)255);
}

int lifted_gram(const double *UX, int64_t nx, int64_t lx, const double *UY, int64_t ny,
                int64_t ly, int64_t width, const int64_t *slot_offsets, int M, int order,
                int difference, int norm, int symmetric, int64_t row_begin, int64_t row_end,
                const double *diag_x, const double *diag_y, double *K, int64_t ldk,
                double *levels, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (symmetric) {
    UY = UX;
    ny = nx;
    ly = lx;
  }
  GenParams P = lifted_base(UX, nx, lx, UY, ny, ly, width, difference);
  if (int e = lifted_params(P, slot_offsets, M, order)) return e;
  P.mode = symmetric ? 1 : 0;
  if (row_end <= row_begin || ny <= 0) return SK_OK;
  // Slot Grams precomputed by block of x rows when the workspace holds them
  // (sk_lifted_gram_workspace_bytes); otherwise inner products on the fly.
  const int64_t bx = g_block_rows(nx, lx, ny, ly, M);
  const size_t g_bytes = (size_t)M * bx * lx * ny * ly * sizeof(double);
  const size_t dp_bytes = lifted_workspace_bytes(bx * ny, ly, M, order, difference);
  if (M < 1 || !ws || ws_bytes < dp_bytes + ((g_bytes + 255) & ~(size_t)255)) {
    P.row_begin = row_begin;
    return run_chunks(P, (row_end - row_begin) * ny, norm, diag_x, diag_y, K, ldk, levels,
                      nullptr, ws, ws_bytes, st);
  }
  double *G = (double *)((char *)ws + ((dp_bytes + 255) & ~(size_t)255));
  P.G = G;
  P.g_ld = ny * ly;
  P.g_lvl = bx * lx * ny * ly;
  for (int64_t b0 = row_begin; b0 < row_end; b0 += bx) {
    const int64_t b1 = std::min(row_end, b0 + bx), rows = (b1 - b0) * lx, cols = ny * ly;
    for (int h = 0; h < M; ++h) {
      const int w = P.woff[h + 1] - P.woff[h];
      const dim3 grid((unsigned)((cols + DG_T - 1) / DG_T), (unsigned)((rows + DG_T - 1) / DG_T));
      dgemm_nt_kernel<<<grid, 256, 0, st>>>(UX + b0 * lx * width + P.woff[h], width,
                                            UY + P.woff[h], width, rows, cols, w,
                                            G + h * P.g_lvl, P.g_ld);
      SK_CHECK_LAUNCH();
    }
    P.g_row0 = b0;
    P.row_begin = b0;
    GenParams Q = P;
    int rc;
    if (symmetric) {
      rc = run_chunks(Q, (b1 - b0) * ny, norm, diag_x, diag_y, K, ldk, levels, nullptr, ws,
                      dp_bytes, st);
    } else {
      // cross: K / levels rows are relative to the caller's row_begin
      rc = run_chunks(Q, (b1 - b0) * ny, norm, diag_x, diag_y,
                      K ? K + (b0 - row_begin) * ldk : nullptr, ldk,
                      levels ? levels + (b0 - row_begin) * ldk * (M + 1) : nullptr, nullptr, ws,
                      dp_bytes, st);
    }
    if (rc) return rc;
  }
  return SK_OK;
}

int lifted_self_levels(const double *UX, int64_t n, int64_t l, int64_t width,
                       const int64_t *slot_offsets, int M, int order, int difference,
                       double *out, void *ws, size_t ws_bytes, cudaStream_t st) {
  GenParams P = lifted_base(UX, n, l, UX, n, l, width, difference);
  if (int e = lifted_params(P, slot_offsets, M, order)) return e;
  P.mode = 2;
  if (n <= 0) return SK_OK;
  // per-sequence slot Grams by a batched float64 GEMM when the workspace holds
  // them (sk_lifted_gram_workspace_bytes(n, l, 1, l, ...)), else on the fly
  const size_t dp_bytes = lifted_workspace_bytes(n, l, M, order, difference);
  const size_t g_bytes = (size_t)M * n * l * l * sizeof(double);
  if (M >= 1 && ws && ws_bytes >= dp_bytes + ((g_bytes + 255) & ~(size_t)255) &&
      n <= 65535) {
    double *G = (double *)((char *)ws + ((dp_bytes + 255) & ~(size_t)255));
    P.G = G;
    P.g_ld = l;
    P.g_lvl = n * l * l;
    for (int h = 0; h < M; ++h) {
      const int w = P.woff[h + 1] - P.woff[h];
      const dim3 grid((unsigned)((l + DG_T - 1) / DG_T), (unsigned)((l + DG_T - 1) / DG_T),
                      (unsigned)n);
      dgemm_nt_kernel<<<grid, 256, 0, st>>>(UX + P.woff[h], width, UX + P.woff[h], width, l, l, w,
                                            G + h * P.g_lvl, l, l * width, l * width, l * l);
      SK_CHECK_LAUNCH();
    }
    return run_chunks(P, n, SK_NORM_NONE, nullptr, nullptr, nullptr, 0, nullptr, out, ws,
                      dp_bytes, st);
  }
  return run_chunks(P, n, SK_NORM_NONE, nullptr, nullptr, nullptr, 0, nullptr, out, ws,
                    ws_bytes, st);
}

size_t generic_levels_dp_workspace_bytes(int64_t batch, int64_t t2, int M, int p) {
  p = std::max(1, std::min(p, std::max(M, 1)));
  return (size_t)std::max<int64_t>(batch, 1) * (scratch_slots(t2, 0, M, p) + M + 1) *
         sizeof(double);
}

int generic_levels_from_increments(const double *A, int64_t batch, int64_t t1, int64_t t2,
                                   int M, int p, int per_level, double *out, void *ws,
                                   size_t ws_bytes, cudaStream_t st) {
  if (batch <= 0) return SK_OK;
  GenParams P{};
  P.A = A;
  P.M = M;
  P.p = std::max(1, std::min(p, std::max(M, 1)));
  P.per_level = per_level;
  P.mode = 3;
  P.t1 = t1;
  P.t2 = t2;
  P.ly = 0;
  P.nx = P.ny = batch;
  P.difference = 1;
  // the per-level layout indexes A with the full batch, so the batch is one chunk
  const size_t need = generic_levels_dp_workspace_bytes(batch, t2, M, P.p);
  if (ws == nullptr || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small for sk_levels_dp: need " +
                                      std::to_string(need) + " bytes");
  const int64_t slots = scratch_slots(t2, 0, M, P.p);
  P.scratch = (double *)ws;
  P.lv = P.scratch + batch * slots;
  P.g0 = 0;
  P.count = batch;
  const int blocks = (int)((batch + GEN_THREADS - 1) / GEN_THREADS);
  generic_levels_kernel<<<blocks, GEN_THREADS, 0, st>>>(P);
  SK_CHECK_LAUNCH();
  const int64_t n = batch * (M + 1);
  copy_levels_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(P.lv, batch, M, out);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

// ---------------------------------------------------------------------------
// increment_tensor (kernels.py:263-281), float64.
// ---------------------------------------------------------------------------
namespace {
__global__ void increment_kernel(const double *X, int64_t nx, int64_t lx, const double *Y,
                                 int64_t ny, int64_t ly, int64_t d, int paired, StaticF64 S,
                                 int difference, int64_t t1, int64_t t2, double *out) {
  const int64_t npairs = paired ? nx : nx * ny;
  const int64_t total = npairs * t1 * t2;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e % t2;
    const int64_t r = (e / t2) % t1;
    const int64_t g = e / (t1 * t2);
    const int64_t i = paired ? g : g / ny;
    const int64_t j = paired ? g : g % ny;
    const double *xs = X + i * lx * d;
    const double *ys = Y + j * ly * d;
    double v;
    if (difference) {
      const double g11 = static_eval_f64(S, xs + (r + 1) * d, ys + (c + 1) * d, (int)d);
      const double g01 = static_eval_f64(S, xs + r * d, ys + (c + 1) * d, (int)d);
      const double g10 = static_eval_f64(S, xs + (r + 1) * d, ys + c * d, (int)d);
      const double g00 = static_eval_f64(S, xs + r * d, ys + c * d, (int)d);
      v = g11 - g01 - g10 + g00;
    } else {
      v = static_eval_f64(S, xs + r * d, ys + c * d, (int)d);
    }
    out[e] = v;
  }
}
}  // namespace

int increment_tensor(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                     int64_t ly, int64_t d, int paired, const sk_static_spec &sp,
                     int difference, double *out, cudaStream_t st) {
  const int64_t t1 = difference ? std::max<int64_t>(lx - 1, 0) : lx;
  const int64_t t2 = difference ? std::max<int64_t>(ly - 1, 0) : ly;
  const int64_t total = (paired ? nx : nx * ny) * t1 * t2;
  if (total <= 0) return SK_OK;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
  increment_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, nx, lx, Y, ny, ly, d, paired,
                                                     to_static(sp), difference, t1, t2, out);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

// Upper-triangle pairwise distances for median_heuristic (static/kernels.py:165-187).
__global__ void pairwise_dist_kernel(const double *__restrict__ X, int64_t n, int64_t d,
                                     double *__restrict__ out) {
  const int64_t npairs = n * (n - 1) / 2;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < npairs;
       t += (int64_t)gridDim.x * blockDim.x) {
    // row i holds n-1-i pairs starting at off(i) = i*(2n-i-1)/2
    int64_t i = (int64_t)((2.0 * n - 1.0 - sqrt((2.0 * n - 1.0) * (2.0 * n - 1.0) - 8.0 * t)) / 2.0);
    while (i > 0 && i * (2 * n - i - 1) / 2 > t) --i;
    while ((i + 1) * (2 * n - i - 2) / 2 <= t) ++i;
    const int64_t j = t - i * (2 * n - i - 1) / 2 + i + 1;
    const double *x = X + i * d, *y = X + j * d;
    double xx = 0.0, yy = 0.0, xy = 0.0;
    for (int64_t k = 0; k < d; ++k) {
      xx = fma(x[k], x[k], xx);
      yy = fma(y[k], y[k], yy);
      xy = fma(x[k], y[k], xy);
    }
    double sq = xx + yy - 2.0 * xy;
    out[t] = sqrt(sq > 0.0 ? sq : 0.0);
  }
}

int pairwise_dist(const double *X, int64_t n, int64_t d, double *out, cudaStream_t st) {
  const int64_t npairs = n * (n - 1) / 2;
  if (npairs <= 0) return SK_OK;
  const int64_t blocks = std::min<int64_t>((npairs + 255) / 256, (int64_t)sm_count() * 32);
  pairwise_dist_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, n, d, out);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

}  // namespace sk
