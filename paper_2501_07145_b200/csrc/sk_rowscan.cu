// Float64 level recursion at order p = 1 with one CTA per sequence pair.
//
// The reference's recursion (kernels.py:174-199 at p = 1: R_m = A * S(R_{m-1}),
// S the 2-D exclusive prefix) is streamed row by row over the pair's T1 x T2
// increment grid, the columns split into contiguous blocks over the CTA's 256
// threads. Per row every thread forms its cells' increments from the float64
// point kernel (the left-boundary point-kernel value comes from the previous
// thread: shuffle, or shared memory across warps), takes the exclusive row
// prefix of every level's column accumulators with one block-wide scan of
// M-1 values, and updates the level sums. Column accumulators live in a
// per-CTA global scratch slice (L2-resident, (M-1) x T2 doubles).
//
// This replaces the thread-per-pair float64 kernel (sk_generic.cu) where one
// pair must be fast: the certification fix-ups of the FP32 paths (a flagged
// c3 entry costs ~0.6 s on the thread-per-pair kernel, a c5 entry ~17 s,
// because a lone thread walks the grid through dependent global-memory state)
// and the order-1 float64 Gram.
#include <algorithm>

#include "sk_common.cuh"

namespace sk {
namespace rowscan {

constexpr int RT = 256;            // threads per CTA
constexpr int NW = RT / 32;
constexpr int CMAX = 16;           // columns per thread: T2 <= 4096 (cta_pair_levels_t)
constexpr int VMAX = GEN_MAX_LEVELS - 1;  // scanned levels (1..M-1)
// channel count above which the point kernel is a block DGEMM (the cells of
// 16-row blocks, or of a whole short pair) instead of per-cell dot products:
// rbf at d = 24 ran 3x slower per cell than at d = 40 on the per-cell form
constexpr int WIDE_D = 16;
constexpr int YSTAGE_BYTES = 96 * 1024;   // dynamic shared memory: y staging / wide blocks
constexpr int WR = 16, KW = 16;           // wide path: point-kernel rows per block, channels per stage
constexpr int WIDE_COLS = (YSTAGE_BYTES / 8 - WR * KW - RT * (KW + 1)) / WR;  // max columns of a block
__device__ __forceinline__ int64_t ystage_doubles() { return YSTAGE_BYTES / 8; }
__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}
constexpr int DYN_SMEM_MAX = 200 * 1024;  // long-row launches: staged y + column state

// The static kernel evaluations of this file are out-of-line calls: inlined
// into every unrolled instance they made ptxas take over ten minutes.
// y's channels ystride apart (1: a point-major row; ly: the channel-major staging)
__device__ __noinline__ double kf_eval(const StaticF64 &S, const double *x, const double *y,
                                       int64_t ystride, int d) {
  double xy = 0.0, xx = 0.0, yy = 0.0;
  for (int k = 0; k < d; ++k) {
    const double yv = y[k * ystride];
    xy = fma(x[k], yv, xy);
    xx = fma(x[k], x[k], xx);
    yy = fma(yv, yv, yy);
  }
  if (S.kind == SK_LINEAR || S.kind == SK_POLYNOMIAL) return static_from_inner(S, xy);
  return static_from_sq(S, xx + yy - 2.0 * xy);  // static_eval_f64's formula
}
__device__ __noinline__ double kf_sq(const StaticF64 &S, double sq) {
  return static_from_sq(S, sq);
}
__device__ __noinline__ double kf_inner(const StaticF64 &S, double xy) {
  return static_from_inner(S, xy);
}
// out[r * WIDE_COLS] = k(v[r]) for a block column (one call for WR / 2 values)
constexpr int WR_ = 16;
__device__ __noinline__ void kf_many(const StaticF64 &S, bool inner, const double (&v)[WR_ / 2],
                                     double *out);

struct Geo {
  const double *X, *Y;
  int64_t nx, lx, ny, ly, d;
  StaticF64 S;
  int M, difference;
};

// Block-wide exclusive prefix of nv values per thread (in place); every thread
// must call it. sm: NW * VMAX doubles.
template <int NVB>
__device__ __forceinline__ void block_excl_scan(double (&v)[NVB], int nv, double *sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double inc[NVB];
#pragma unroll
  for (int k = 0; k < NVB; ++k) inc[k] = v[k];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int k = 0; k < NVB; ++k) {
      if (k < nv) {
        const double u = __shfl_up_sync(0xffffffffu, inc[k], o);
        if (lane >= o) inc[k] += u;
      }
    }
  }
  if (lane == 31)
    for (int k = 0; k < nv; ++k) sm[warp * VMAX + k] = inc[k];
  __syncthreads();
  for (int k = 0; k < nv; ++k) {
    double off = 0.0;
    for (int w = 0; w < warp; ++w) off += sm[w * VMAX + k];
    v[k] = off + inc[k] - v[k];
  }
  __syncthreads();  // sm reusable
}

// Block-wide sum of v[0..n) into out[0..n) (thread 0). sm: NW * (VMAX + 1).
__device__ __forceinline__ void block_sum(const double *v, int n, double *sm, double *out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < n; ++k) {
    double s = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sm[warp * (VMAX + 1) + k] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < n; ++k) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += sm[w * (VMAX + 1) + k];
      out[k] = s;
    }
  __syncthreads();
}

static_assert(WR == WR_, "kf_many block height");
__device__ __noinline__ void kf_many(const StaticF64 &S, bool inner, const double (&v)[WR_ / 2],
                                     double *out) {
  for (int r = 0; r < WR_ / 2; ++r)
    out[r * WIDE_COLS] = inner ? static_from_inner(S, v[r]) : static_from_sq(S, v[r]);
}

// Point-kernel rows gb .. gb+rb of the pair into gblk[r * WIDE_COLS + c],
// c < ncol: a float64 block product of the rows' x points and all y points,
// KW channels per shared-memory stage (thread = column, WR accumulators).
__device__ __noinline__ void wide_block(const Geo &G, const double *__restrict__ xs,
                                        const double *__restrict__ ys, int64_t gb, int rb,
                                        int64_t ncol, double *gblk) {
  // two threads per column, RPT rows each: 128 columns per pass
  constexpr int RPT = WR / 2, CPP = RT / 2;
  const int t = threadIdx.x, d = (int)G.d;
  const int ct = t >> 1, r0 = (t & 1) * RPT;
  const bool inner = G.S.kind == SK_LINEAR || G.S.kind == SK_POLYNOMIAL;
  double *xt = gblk + WR * WIDE_COLS, *yt = xt + WR * KW;
  for (int cb = 0; cb < ncol; cb += CPP) {  // columns c = cb + ct
    const int c = cb + ct;
    double acc[WR_ / 2], xx[WR_ / 2];
#pragma unroll
    for (int r = 0; r < RPT; ++r) acc[r] = xx[r] = 0.0;
    double yy = 0.0;
    // stage loads prefetched one stage ahead into registers (the staging was
    // latency-bound: every shared store waited for its global load)
    constexpr int XE = (WR * KW + RT - 1) / RT, YE = (CPP * KW + RT - 1) / RT;
    double xr[XE], yr[YE];
    auto fetch = [&](int k0) {
      const int kn = d - k0 < KW ? d - k0 : KW;
#pragma unroll
      for (int u = 0; u < XE; ++u) {
        const int e = t + u * RT, r = e / KW, k = e % KW;
        xr[u] = (e < WR * KW && r < rb && k < kn) ? xs[(gb + r) * d + k0 + k] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < YE; ++u) {
        const int e = t + u * RT, cc = e / KW, k = e % KW;
        yr[u] = (e < CPP * KW && cb + cc < ncol && k < kn) ? ys[(int64_t)(cb + cc) * d + k0 + k]
                                                           : 0.0;
      }
    };
    fetch(0);
    for (int k0 = 0; k0 < d; k0 += KW) {
      __syncthreads();  // the previous stage's readers are done
#pragma unroll
      for (int u = 0; u < XE; ++u)
        if (t + u * RT < WR * KW) xt[t + u * RT] = xr[u];
#pragma unroll
      for (int u = 0; u < YE; ++u) {  // rows padded to KW + 1: conflict-free column reads
        const int e = t + u * RT;
        if (e < CPP * KW) yt[(e / KW) * (KW + 1) + e % KW] = yr[u];
      }
      __syncthreads();
      if (k0 + KW < d) fetch(k0 + KW);
      if (inner) {
#pragma unroll
        for (int k = 0; k < KW; ++k) {
          const double yv = yt[ct * (KW + 1) + k];
#pragma unroll
          for (int r = 0; r < RPT; ++r) acc[r] = fma(xt[(r0 + r) * KW + k], yv, acc[r]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < KW; ++k) {
          const double yv = yt[ct * (KW + 1) + k];
          yy = fma(yv, yv, yy);
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const double xv = xt[(r0 + r) * KW + k];
            acc[r] = fma(xv, yv, acc[r]);
            xx[r] = fma(xv, xv, xx[r]);
          }
        }
      }
    }
    if (c < ncol) {
      if (!inner)
#pragma unroll
        for (int r = 0; r < RPT; ++r) acc[r] = xx[r] + yy - 2.0 * acc[r];
      if (G.S.kind == SK_LINEAR) {  // inline: no call per output
#pragma unroll
        for (int r = 0; r < RPT; ++r) gblk[(r0 + r) * WIDE_COLS + c] = G.S.scale * acc[r];
      } else {
        kf_many(G.S, inner, acc, gblk + r0 * WIDE_COLS + c);
      }
    }
  }
  __syncthreads();
}

// Level values k_0..k_M of the pair (xs: lx points, ys: ly points) into
// lv_out[0..M] (shared memory, written by thread 0; visible after return).
// colacc: this CTA's scratch slice (slot_doubles). All threads call it.
// CC: compile-time columns per thread (>= ceil(T2 / RT)); every per-thread
// array is indexed by unrolled compile-time loops so it stays in registers.
template <int CC, int MB>
__device__ __noinline__ void cta_pair_levels_t(const Geo &G, const double *__restrict__ xs, int64_t lx,
                                  const double *ys, int64_t ly, double *__restrict__ colacc,
                                  double *sm, double *lv_out) {
  const int M = G.M, d = (int)G.d;
  const int64_t T1 = G.difference ? lx - 1 : lx, T2 = G.difference ? ly - 1 : ly;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int C = (int)((T2 + RT - 1) / RT);
  const int64_t c0 = std::min<int64_t>((int64_t)t * C, T2);
  const int n = (int)(std::min<int64_t>(c0 + C, T2) - c0);  // own cells of a row
  const int NV = M - 1;
  // column accumulators of levels 1..M-1 for the own columns: registers for
  // CC <= 2 (every loop unrolled), else the scratch slice (rows of T2 doubles)
  constexpr bool REG = CC <= 2;
  constexpr int VB = MB - 1;  // level bound of this instance (M <= MB)
  double ca[REG ? VB : 1][REG ? CC : 1];
  // MEM variant: the scratch slice after the row buffer ([m][column]), or
  // shared memory after the staged y sequence when the launch gave enough
  // ([m][k][thread], conflict-free) — L2 round trips per level and row were
  // the long-row kernel's bound (c5 pair: 68 ms, 67% long-scoreboard stalls)
  double *cm_base = colacc + T2 + 2 + c0;
  int64_t cm_sm = T2, cm_sk = 1;
  auto CA = [&](int m, int k) -> double & {
    if constexpr (REG) return ca[m][k];
    else return cm_base[m * cm_sm + k * cm_sk];
  };
  double lsum[MB], tot[VB];
#pragma unroll
  for (int m = 0; m < MB; ++m) lsum[m] = 0.0;
#pragma unroll
  for (int m = 0; m < VB; ++m) tot[m] = 0.0;
  double *smb = sm + NW * VMAX;  // warp-boundary point-kernel values
  // d > WIDE_D: a row's point-kernel values are formed warp-cooperatively (lanes
  // over channels: coalesced reads of every y point) into a row buffer in the
  // scratch slice; otherwise every thread evaluates its own columns
  const bool wide = d > WIDE_D;
  double *grow = colacc;
  const bool inner = G.S.kind == SK_LINEAR || G.S.kind == SK_POLYNOMIAL;
  const int64_t ncol = G.difference ? T2 + 1 : T2;
  // narrow rows read every y point once per row: stage the pair's y sequence
  // in shared memory when it fits (ystage_doubles), else read it from L1/L2
  // (channel-major: point c's channel k at [k * ly + c], so the threads of a
  // warp read consecutive addresses — point-major put them 8 d bytes apart,
  // all in one shared-memory bank)
  extern __shared__ double ystage[];
  int64_t ysc = d, ysk = 1;  // strides of point / channel in ys
  if (!wide && ly * d <= ystage_doubles()) {
    __syncthreads();  // the previous pair's readers are done
    for (int64_t e = t; e < ly * d; e += RT) ystage[(e % d) * ly + e / d] = ys[e];
    __syncthreads();
    ys = ystage;
    ysc = 1;
    ysk = ly;
    if constexpr (!REG) {
      const int64_t off = (ly * d + 1) & ~(int64_t)1;
      if ((off + (int64_t)NV * C * RT) * 8 <= (int64_t)dyn_smem_bytes()) {
        cm_base = ystage + off + t;
        cm_sm = (int64_t)C * RT;
        cm_sk = RT;
      }
    }
  }
  if constexpr (REG) {
#pragma unroll
    for (int m = 0; m < VB; ++m)
#pragma unroll
      for (int k = 0; k < CC; ++k) ca[m][k] = 0.0;
  } else {
    for (int m = 0; m < NV; ++m)
#pragma unroll
      for (int k = 0; k < CC; ++k)
        if (k < n) CA(m, k) = 0.0;
  }
  auto yp = [&](int64_t c) { return ys + c * ysc; };
  auto wide_row = [&](const double *xa) {  // grow[c] = k(xa, y_c), c < ncol
    for (int64_t cb = (int64_t)warp * 4; cb < ncol; cb += NW * 4) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = lane; k < d; k += 32) {
        const double xv = xa[k];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (cb + u < ncol) {
            const double yv = ys[(cb + u) * d + k];
            acc[u] = inner ? fma(xv, yv, acc[u]) : fma(xv - yv, xv - yv, acc[u]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
        if (lane == 0 && cb + u < ncol)
          grow[cb + u] = inner ? kf_inner(G.S, acc[u]) : kf_sq(G.S, acc[u]);
      }
    }
    __syncthreads();
  };
  // one row of the level recursion (R_1 = A, R_{m+1} = A * S_m) from this
  // thread's cells a[0..n)
  auto dp_row = [&](const double (&a)[CC]) {
    // exclusive row prefix of the column accumulators (old values), levels 1..M-1
    double pre[VB];
#pragma unroll
    for (int m = 0; m < VB; ++m) {
      pre[m] = 0.0;
      if constexpr (REG) {
#pragma unroll
        for (int k = 0; k < CC; ++k) pre[m] += CA(m, k);
      } else {
        pre[m] = tot[m];  // the own columns' total, kept in registers
      }
    }
    block_excl_scan(pre, NV, sm);
    if constexpr (REG) {
#pragma unroll
      for (int k = 0; k < CC; ++k) {
        double Rprev = a[k];  // R_1 (0 beyond the own cells)
        lsum[0] += Rprev;
#pragma unroll
        for (int m = 1; m < MB; ++m) {  // R_{m+1} = A * S_m
          if (m < M) {
            const double R = a[k] * pre[m - 1];
            lsum[m] += R;
            double &acc = CA(m - 1, k);
            const double old = acc;
            pre[m - 1] += old;
            acc = old + Rprev;
            Rprev = R;
          }
        }
      }
    } else {
      // long rows (column state in the scratch slice): level-outer order, so
      // each level's CC accumulators are loaded and stored as one batch of
      // independent accesses (cell-outer order chained (M-1) CC dependent
      // global round trips per row)
      double R[CC];
#pragma unroll
      for (int k = 0; k < CC; ++k) {
        R[k] = k < n ? a[k] : 0.0;  // R_1
        lsum[0] += R[k];
      }
#pragma unroll
      for (int m = 1; m < MB; ++m) {
        if (m < M) {
          double cav[CC];
#pragma unroll
          for (int k = 0; k < CC; ++k) cav[k] = k < n ? CA(m - 1, k) : 0.0;
          double p = pre[m - 1], rs = 0.0;
#pragma unroll
          for (int k = 0; k < CC; ++k) {
            const double Rn = a[k] * p;  // R_{m+1}, S_m = the prefix left of column k
            lsum[m] += Rn;               // a[k] = 0 beyond the own cells
            p += cav[k];
            cav[k] += R[k];
            rs += R[k];
            R[k] = Rn;
          }
          tot[m - 1] += rs;
#pragma unroll
          for (int k = 0; k < CC; ++k)
            if (k < n) CA(m - 1, k) = cav[k];
        }
      }
    }
  };
  // point-kernel values of the previous row at columns c0 .. c0 + n (difference)
  double gp[CC + 1];
  if (wide && ncol <= WIDE_COLS) {
    // Row blocks of WR point-kernel rows at a time: a float64 block product of
    // the block's x points and all y points, KW channels per shared-memory
    // stage (thread = column, WR accumulators), into gblk[WR][ncol]; the
    // recursion then reads its rows from shared memory.
    double *gblk = ystage;
    const int64_t nrows = G.difference ? lx : T1;  // point-kernel rows
    for (int64_t gb = 0; gb < nrows; gb += WR) {
      const int rb = nrows - gb < WR ? (int)(nrows - gb) : WR;
      wide_block(G, xs, ys, gb, rb, ncol, gblk);
      __syncthreads();
      for (int r = 0; r < rb; ++r) {
        const double *grow_s = gblk + r * WIDE_COLS;
        double a[CC];
        if (G.difference) {
          double g[CC + 1];
#pragma unroll
          for (int k = 0; k <= CC; ++k) g[k] = k <= n ? grow_s[c0 + k] : 0.0;
          if (gb + r > 0) {
            // kernels.py:281: G[1:,1:] - G[:-1,1:] - G[1:,:-1] + G[:-1,:-1]
#pragma unroll
            for (int k = 0; k < CC; ++k)
              a[k] = k < n ? g[k + 1] - gp[k + 1] - g[k] + gp[k] : 0.0;
          }
#pragma unroll
          for (int k = 0; k <= CC; ++k) gp[k] = g[k];
          if (gb + r == 0) continue;  // point row 0: no increment row yet (CTA-uniform)
        } else {
#pragma unroll
          for (int k = 0; k < CC; ++k) a[k] = k < n ? grow_s[c0 + k] : 0.0;
        }
        dp_row(a);
      }
    }
  } else {
    if (G.difference) {
      if (wide) {
        wide_row(xs);
#pragma unroll
        for (int k = 0; k <= CC; ++k) gp[k] = k <= n ? grow[c0 + k] : 0.0;
        __syncthreads();
      } else {
#pragma unroll
        for (int k = 0; k <= CC; ++k)
          gp[k] = k <= n ? kf_eval(G.S, xs, yp(c0 + k), ysk, d) : 0.0;
      }
    }
    for (int64_t r = 0; r < T1; ++r) {
      double a[CC];
      if (G.difference) {
        const double *xa = xs + (r + 1) * d;
        double g[CC + 1];
        if (wide) {
          wide_row(xa);
#pragma unroll
          for (int k = 0; k <= CC; ++k) g[k] = k <= n ? grow[c0 + k] : 0.0;
          __syncthreads();  // grow is rewritten next row
        } else {
          // G(r+1, c0 + k) for k = 1..n here; k = 0 from the previous thread
#pragma unroll
          for (int k = 1; k <= CC; ++k)
            g[k] = k <= n ? kf_eval(G.S, xa, yp(c0 + k), ysk, d) : 0.0;
          double last = 0.0;
#pragma unroll
          for (int k = 1; k <= CC; ++k)
            if (k == n) last = g[k];
          const double up = __shfl_up_sync(0xffffffffu, last, 1);
          if (lane == 31) smb[warp] = last;
          __syncthreads();
          if (t == 0)
            g[0] = kf_eval(G.S, xa, yp(0), ysk, d);
          else
            g[0] = lane == 0 ? smb[warp - 1] : up;
        }
        // kernels.py:281: G[1:,1:] - G[:-1,1:] - G[1:,:-1] + G[:-1,:-1]
#pragma unroll
        for (int k = 0; k < CC; ++k) a[k] = k < n ? g[k + 1] - gp[k + 1] - g[k] + gp[k] : 0.0;
#pragma unroll
        for (int k = 0; k <= CC; ++k) gp[k] = g[k];
      } else if (wide) {
        wide_row(xs + r * d);
#pragma unroll
        for (int k = 0; k < CC; ++k) a[k] = k < n ? grow[c0 + k] : 0.0;
        __syncthreads();
      } else {
#pragma unroll
        for (int k = 0; k < CC; ++k)
          a[k] = k < n ? kf_eval(G.S, xs + r * d, yp(c0 + k), ysk, d) : 0.0;
      }
      dp_row(a);
    }
  }
  block_sum(lsum, M, sm, lv_out + 1);
  if (t == 0) lv_out[0] = 1.0;
  __syncthreads();
}

__device__ __noinline__ void cta_pair_levels(const Geo &G, const double *__restrict__ xs, int64_t lx,
                                const double *__restrict__ ys, int64_t ly,
                                double *__restrict__ colacc, double *sm, double *lv_out) {
  const int64_t T1 = G.difference ? lx - 1 : lx, T2 = G.difference ? ly - 1 : ly;
  if (G.M == 0 || T1 <= 0 || T2 <= 0) {
    if (threadIdx.x == 0) {
      lv_out[0] = 1.0;
      for (int m = 1; m <= G.M; ++m) lv_out[m] = 0.0;
    }
    __syncthreads();
    return;
  }
  // instances: columns per thread x level bound (M <= 4 / 8 / 16)
  const int64_t C = (T2 + RT - 1) / RT;
  const int M = G.M;
#define SK_RS(CCV, MBV) cta_pair_levels_t<CCV, MBV>(G, xs, lx, ys, ly, colacc, sm, lv_out)
  if (C <= 1) {
    if (M <= 4) SK_RS(1, 4); else if (M <= 8) SK_RS(1, 8); else SK_RS(1, 16);
  } else if (C <= 2) {
    if (M <= 4) SK_RS(2, 4); else if (M <= 8) SK_RS(2, 8); else SK_RS(2, 16);
  } else if (C <= 8) {
    if (M <= 8) SK_RS(8, 8); else SK_RS(8, 16);
  } else {
    SK_RS(16, 16);
  }
#undef SK_RS
}

// --- wide short pairs (d > WIDE_D, L <= 128): block DGEMM + one-warp DP ------
// The redo of the GEMM-fed path's flagged entries (c4: ~6% of a 4096^2 Gram)
// is float64 GEMM work: 2.1 M FMAs per pair at d = 128. One CTA forms the
// pair's whole point-kernel matrix in shared memory with a register-blocked
// float64 product (8 x 8 outputs per thread, 16 channels per stage, the raw
// points of the next stage in flight by cp.async while the current one is
// multiplied), then warp 0 runs the recursion on it, double-differencing on
// read (kernels.py:281; lanes own 4 columns, one warp-level scan per level and
// row, no block barriers).
constexpr int WP = 128;          // max points (rows / columns) of a wide short pair
constexpr int WPS = WP + 1;      // padded row stride of the matrix in shared memory
constexpr int WK = 16;           // channels per stage
constexpr int WKS = WK + 1;
constexpr int WSTAGE = 2 * WP * WKS;  // one stage buffer: x rows then y rows
constexpr size_t WIDE_SMEM = (size_t)(WP * WPS + 2 * WSTAGE + 2 * WP) * 8;

__device__ __forceinline__ void cp_async8(double *smem_dst, const double *gmem_src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit8() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait8() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

bool wide_short(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  const int p = std::max(1, std::min(c.order, std::max(c.n_levels, 1)));
  return p == 1 && d > WIDE_D && lx <= WP && ly <= WP && c.n_levels <= GEN_MAX_LEVELS;
}

// linear kind with differences: wide_point_matrix leaves the raw inner
// products and the double difference applies the scale (the kernel is
// bilinear, kernels.py:281), saving a pass over the matrix
__device__ __forceinline__ double wide_dd_scale(const Geo &G) {
  return G.S.kind == SK_LINEAR && G.difference ? G.S.scale : 1.0;
}

// The pair's point-kernel matrix Am[r][c] = k(x_r, y_c) (r < lx, c < ly) into
// shared memory (row stride WPS; linear with differences: the raw inner
// products, see wide_dd_scale). All threads call it; Am is complete on return.
__device__ __noinline__ void wide_point_matrix(const Geo &G, const double *__restrict__ xs,
                                               int64_t lx, const double *__restrict__ ys,
                                               int64_t ly, double *smem) {
  const int t = threadIdx.x, d = (int)G.d;
  const bool inner = G.S.kind == SK_LINEAR || G.S.kind == SK_POLYNOMIAL;
  const int R = (int)lx, C = (int)ly;  // the point-kernel matrix formed
  double *Am = smem, *stg = Am + WP * WPS, *xn = stg + 2 * WSTAGE, *yn = xn + WP;
  const int ty = t >> 4, tx = t & 15;
  double acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.0;
  double nrm = 0.0;  // |x_r|^2 (t < 128) or |y_c|^2 (t >= 128): stationary kinds
  const auto issue = [&](int k0, double *buf) {
    for (int e = t; e < WP * WK; e += RT) {
      const int r = e / WK, k = e % WK, kk = k0 + k;
      double *xd = buf + r * WKS + k, *yd = buf + WP * WKS + r * WKS + k;
      if (kk < d && r < R) cp_async8(xd, xs + r * d + kk); else *xd = 0.0;
      if (kk < d && r < C) cp_async8(yd, ys + r * d + kk); else *yd = 0.0;
    }
    cp_async_commit8();
  };
  __syncthreads();  // the previous pair's readers of the stage buffers are done
  issue(0, stg);
  for (int s = 0, k0 = 0; k0 < d; ++s, k0 += WK) {
    const double *xt = stg + (s & 1) * WSTAGE, *yt = xt + WP * WKS;
    if (k0 + WK < d) {
      issue(k0 + WK, stg + ((s + 1) & 1) * WSTAGE);
      cp_async_wait8<1>();
    } else {
      cp_async_wait8<0>();
    }
    __syncthreads();
    if (!inner) {
      const double *row = t < WP ? xt + t * WKS : yt + (t - WP) * WKS;
#pragma unroll
      for (int k = 0; k < WK; ++k) nrm = fma(row[k], row[k], nrm);
    }
#pragma unroll 4
    for (int k = 0; k < WK; ++k) {
      double xv[8], yv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = xt[(ty + 16 * u) * WKS + k];
#pragma unroll
      for (int v = 0; v < 8; ++v) yv[v] = yt[(tx + 16 * v) * WKS + k];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fma(xv[u], yv[v], acc[u][v]);
    }
    __syncthreads();  // this buffer is refilled two stages on
  }
  if (!inner) (t < WP ? xn[t] : yn[t - WP]) = nrm;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int r = ty + 16 * u, c = tx + 16 * v;
      if (r < R && c < C) Am[r * WPS + c] = inner ? acc[u][v] : xn[r] + yn[c] - 2.0 * acc[u][v];
    }
  __syncthreads();
  // the static kernel in a rolled loop: one copy of its code (inlined into the
  // unrolled tile above it was 64 copies, and the instruction cache missed)
  const StaticF64 S = G.S;
  if (S.kind == SK_LINEAR && G.difference) return;  // scale applied by the double difference
  for (int r = t / WP; r < R; r += RT / WP) {
    const int c = t % WP;
    if (c < C) {
      double &v = Am[r * WPS + c];
      v = inner ? static_from_inner(S, v) : static_from_sq(S, v);
    }
  }
  __syncthreads();
}

// The order-1 recursion of one pair by one warp on a matrix a(i, c) (i < T1,
// c < T2 <= 128): lanes own 4 columns, one warp-level exclusive scan per level
// and row (kernels.py:144-201). Lane 0 writes lv_out[0..M].
template <int MB, class F>
__device__ __forceinline__ void warp_levels(F a_of, int T1, int T2, int M, int lane,
                                            double *lv_out) {
  constexpr int VB = MB - 1;
  double ca[VB > 0 ? VB : 1][4], lsum[MB];
#pragma unroll
  for (int m = 0; m < VB; ++m)
#pragma unroll
    for (int k = 0; k < 4; ++k) ca[m][k] = 0.0;
#pragma unroll
  for (int m = 0; m < MB; ++m) lsum[m] = 0.0;
  const int c0 = 4 * lane;
  // rows are read two ahead: the batched redo's matrices come from L2, and
  // the recursion is one serial chain per warp
  double nx1[4], nx2[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    nx1[k] = c0 + k < T2 ? a_of(0, c0 + k) : 0.0;
    nx2[k] = 1 < T1 && c0 + k < T2 ? a_of(1, c0 + k) : 0.0;
  }
  for (int i = 0; i < T1; ++i) {
    double a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[k] = nx1[k];
      nx1[k] = nx2[k];
      nx2[k] = i + 2 < T1 && c0 + k < T2 ? a_of(i + 2, c0 + k) : 0.0;
    }
    // exclusive prefix over columns of every level's accumulators (old values)
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
      double Rprev = a[k];
      lsum[0] += Rprev;
#pragma unroll
      for (int m = 1; m < MB; ++m) {
        if (m < M) {
          const double Rn = a[k] * pre[m - 1];
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
    lv_out[0] = 1.0;
#pragma unroll
    for (int m = 0; m < MB; ++m)
      if (m < M) lv_out[m + 1] = lsum[m];
  }
}

// Level values of one pair into lv_out (written by thread 0, visible after return).
template <int MB>
__device__ __noinline__ void wide_pair_levels(const Geo &G, const double *__restrict__ xs,
                                              int64_t lx, const double *__restrict__ ys,
                                              int64_t ly, double *smem, double *lv_out) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, M = G.M;
  const int T1 = (int)(G.difference ? lx - 1 : lx), T2 = (int)(G.difference ? ly - 1 : ly);
  if (M == 0 || T1 <= 0 || T2 <= 0) {
    if (t == 0) {
      lv_out[0] = 1.0;
      for (int m = 1; m <= M; ++m) lv_out[m] = 0.0;
    }
    __syncthreads();
    return;
  }
  wide_point_matrix(G, xs, lx, ys, ly, smem);
  const double *Am = smem;
  const bool diff = G.difference;
  const double sc = wide_dd_scale(G);
  if (warp == 0)
    warp_levels<MB>(
        [&](int i, int c) {
          return diff ? sc * (Am[(i + 1) * WPS + c + 1] - Am[i * WPS + c + 1] -
                              Am[(i + 1) * WPS + c] + Am[i * WPS + c])
                      : Am[i * WPS + c];
        },
        T1, T2, M, lane, lv_out);
  __syncthreads();
}

__device__ __noinline__ void wide_levels(const Geo &G, const double *xs, int64_t lx,
                                         const double *ys, int64_t ly, double *smem,
                                         double *lv_out) {
  if (G.M <= 4)
    wide_pair_levels<4>(G, xs, lx, ys, ly, smem, lv_out);
  else if (G.M <= 8)
    wide_pair_levels<8>(G, xs, lx, ys, ly, smem, lv_out);
  else
    wide_pair_levels<16>(G, xs, lx, ys, ly, smem, lv_out);
}

// --- the order-1 float64 Gram / self levels ---------------------------------
struct GramArgs {
  Geo G;
  int mode;  // 0 rect pairs (rows [row_begin, row_end)), 1 symmetric (j >= i), 2 self
  int64_t row_begin, rows;
  int norm;
  const double *diag_x, *diag_y;
  double *K;
  int64_t ldk;
  double *levels;
  double *self_out;
  double *scratch;
  int64_t slot;  // doubles of scratch per CTA
};

template <bool WIDE>
__global__ void __launch_bounds__(RT, WIDE ? 1 : 2) gram_kernel(GramArgs A) {
  __shared__ double sm[NW * (VMAX + 1) + NW + 2 * (GEN_MAX_LEVELS + 1)];
  double *lv = sm + NW * (VMAX + 1) + NW;
  const Geo &G = A.G;
  double *colacc = A.scratch + blockIdx.x * A.slot;
  const int64_t npairs = A.mode == 2 ? G.nx : A.rows * G.ny;
  for (int64_t g = blockIdx.x; g < npairs; g += gridDim.x) {
    int64_t i, j;
    if (A.mode == 2) {
      i = j = g;
    } else {
      i = A.row_begin + g / G.ny;
      j = g % G.ny;
      if (A.mode == 1 && j < i) continue;  // CTA-uniform
    }
    const double *xs = G.X + i * G.lx * G.d;
    const double *ys = (A.mode == 2 ? G.X : G.Y) + j * (A.mode == 2 ? G.lx : G.ly) * G.d;
    if constexpr (WIDE) {
      extern __shared__ double wsm[];
      wide_levels(G, xs, G.lx, ys, A.mode == 2 ? G.lx : G.ly, wsm, lv);
    } else {
      cta_pair_levels(G, xs, G.lx, ys, A.mode == 2 ? G.lx : G.ly, colacc, sm, lv);
    }
    if (threadIdx.x == 0) {
      const int M = G.M;
      if (A.mode == 2) {
        for (int m = 0; m <= M; ++m) A.self_out[i * (M + 1) + m] = lv[m];
      } else {
        const bool sym = A.mode == 1;
        const int64_t row = sym ? i : i - A.row_begin;
        if (A.levels) {
          for (int m = 0; m <= M; ++m) A.levels[(row * A.ldk + j) * (M + 1) + m] = lv[m];
          if (sym && j != i)
            for (int m = 0; m <= M; ++m) A.levels[(j * A.ldk + i) * (M + 1) + m] = lv[m];
        }
        if (A.K) {
          const double v = finish_entry(lv, M, A.norm, A.diag_x ? A.diag_x + i * (M + 1) : nullptr,
                                        A.diag_y ? A.diag_y + j * (M + 1) : nullptr);
          A.K[row * A.ldk + j] = v;
          if (sym && j != i) A.K[j * A.ldk + i] = v;
        }
      }
    }
    __syncthreads();
  }
}

// --- certification of the FP32 paths -----------------------------------------
struct CertArgs {
  Geo G;
  int symmetric;
  int64_t row_begin, rows;
  int norm;
  const double *diag_x, *diag_y;
  const float2 *k1buf;  // per entry [row][ny]: (FP32 level 1, sum_m |k_m|), or null
  int l1check;         // difference=True and n_levels >= 1: the exact-level-1 check
  double *K;
  int64_t ldk;
  double *levels;
  double *scratch;
  int64_t slot;
  // compacted list of the entries the scan flagged: work[0] = count, then the
  // entry indices (row - row_begin) * ny + j; a count above `cap` (or no scan)
  // makes the redo find its entries by scanning K instead
  unsigned long long *work;
  int64_t cap;
};

__device__ __forceinline__ void flag_entry(const CertArgs &A, int64_t e) {
  const unsigned long long q = atomicAdd(A.work, 1ull);
  if ((int64_t)q < A.cap) A.work[1 + q] = (unsigned long long)e;
}

// Pass 1: the exact-level-1 check. The four corner point-kernel values of
// every entry are a small GEMM-shaped contraction over the channels, so CTAs
// take tiles of SR rows x RT columns: the rows' first/last points are staged
// in shared memory (SK channels at a time), every thread streams its column's
// two corner points from the transposed corner arrays (coalesced) and keeps
// 4 SR accumulators. Entries whose FP32 level 1 deviates from the telescoped
// value by more than the tolerance of their scale are marked NaN (with the
// mirror); the others are corrected to the exact level 1.
constexpr int SR = 8, SK = 32;

// Xc[(b * d + k) * n + i] = point (b ? L-1 : 0) of sequence i, channel k
__global__ void corners_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                               double *__restrict__ Xc) {
  const int64_t total = n * 2 * d;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n, rest = t / n, k = rest % d, b = rest / d;
    Xc[t] = X[(i * L + (b ? L - 1 : 0)) * d + k];
  }
}

template <bool INNER>
__global__ void __launch_bounds__(RT) cert_scan_kernel(CertArgs A, const double *__restrict__ Xc,
                                                       const double *__restrict__ Yc) {
  __shared__ double xs[SR][2][SK];
  const Geo &G = A.G;
  const int M = G.M;
  const int d = (int)G.d;
  const bool sym = A.symmetric;
  const int64_t tiles_c = (G.ny + RT - 1) / RT, tiles = ((A.rows + SR - 1) / SR) * tiles_c;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = (tile / tiles_c) * SR, j = (tile % tiles_c) * RT + threadIdx.x;
    const bool jv = j < G.ny;
    double acc[SR][4];
#pragma unroll
    for (int r = 0; r < SR; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.0;
    for (int k0 = 0; k0 < d; k0 += SK) {
      const int kn = min(SK, d - k0);
      for (int e = threadIdx.x; e < SR * 2 * SK; e += RT) {
        const int r = e / (2 * SK), b = (e / SK) & 1, k = e % SK;
        const int64_t i = A.row_begin + r0 + r;
        xs[r][b][k] = (r0 + r < A.rows && k < kn) ? Xc[(b * G.d + k0 + k) * G.nx + i] : 0.0;
      }
      __syncthreads();
      if (jv) {
        for (int k = 0; k < kn; ++k) {
          const double b0 = Yc[(k0 + k) * G.ny + j], b1 = Yc[(G.d + k0 + k) * G.ny + j];
#pragma unroll
          for (int r = 0; r < SR; ++r) {
            const double a0 = xs[r][0][k], a1 = xs[r][1][k];
            if (INNER) {
              acc[r][0] = fma(a0, b0, acc[r][0]);
              acc[r][1] = fma(a0, b1, acc[r][1]);
              acc[r][2] = fma(a1, b0, acc[r][2]);
              acc[r][3] = fma(a1, b1, acc[r][3]);
            } else {
              acc[r][0] = fma(a0 - b0, a0 - b0, acc[r][0]);
              acc[r][1] = fma(a0 - b1, a0 - b1, acc[r][1]);
              acc[r][2] = fma(a1 - b0, a1 - b0, acc[r][2]);
              acc[r][3] = fma(a1 - b1, a1 - b1, acc[r][3]);
            }
          }
        }
      }
      __syncthreads();
    }
    if (!jv) continue;
#pragma unroll
    for (int r = 0; r < SR; ++r) {
      if (r0 + r >= A.rows) break;
      const int64_t i = A.row_begin + r0 + r;
      const int64_t row = sym ? i : r0 + r;
      if (sym && j <= i) continue;  // the diagonal of K(X) is the self levels' own
      double *kp = A.K + row * A.ldk + j;
      const double v = *kp;
      // cancellation beyond what the FP32 levels resolve, or non-finite
      const float2 kv = A.k1buf[row * G.ny + j];
      const double lim = A.norm == SK_NORM_NONE
                             ? (double)kv.y *
                                   (G.S.kind == SK_LINEAR ? CERT_TAU_RAW_LINEAR : CERT_TAU_RAW)
                             : CERT_TAU_NORM;
      if (!(fabs(v) >= lim) || isinf(v)) {
        *kp = __longlong_as_double(0x7ff8000000000000ll);
        if (sym) A.K[j * A.ldk + i] = *kp;
        flag_entry(A, (r0 + r) * G.ny + j);
        continue;
      }
      if (!A.l1check) continue;
      double k1e = 0.0;  // k(x_T,y_T') - k(x_0,y_T') - k(x_T,y_0) + k(x_0,y_0)
      if (G.lx >= 2 && G.ly >= 2) {
        if (INNER)
          k1e = kf_inner(G.S, acc[r][3]) - kf_inner(G.S, acc[r][2]) -
                kf_inner(G.S, acc[r][1]) + kf_inner(G.S, acc[r][0]);
        else
          k1e = kf_sq(G.S, acc[r][3]) - kf_sq(G.S, acc[r][2]) -
                kf_sq(G.S, acc[r][1]) + kf_sq(G.S, acc[r][0]);
      }
      const double delta = k1e - (double)kv.x;
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
      const double nv = fabs(delta) > CERT_NOISE * scale
                            ? __longlong_as_double(0x7ff8000000000000ll)
                            : v + corr;
      *kp = nv;
      if (sym) A.K[j * A.ldk + i] = nv;
      if (isnan(nv)) flag_entry(A, (r0 + r) * G.ny + j);
      if (A.levels && !isnan(nv)) {
        A.levels[(row * A.ldk + j) * (M + 1) + 1] = k1e;
        if (sym) A.levels[(j * A.ldk + i) * (M + 1) + 1] = k1e;
      }
    }
  }
}

// Pass 2: every flagged entry recomputed in float64, one pair (plus both self
// levels when normalised) per CTA. The scan's compacted list is dealt out
// round-robin (every item costs the same, and flagged entries cluster in rows,
// so striding over K itself left most CTAs idle); without a list the CTAs
// stride over the entries RT at a time and collect the NaN ones.
template <bool WIDE>
__device__ void redo_entry(const CertArgs &A, int64_t ee, double *colacc, double *sm,
                           double *lv, double *dx, double *dy) {
  const Geo &G = A.G;
  const int M = G.M;
  const bool sym = A.symmetric;
  const int64_t r = ee / G.ny, j = ee % G.ny, i = A.row_begin + r;
  const int64_t row = sym ? i : r;
  const double *xs = G.X + i * G.lx * G.d, *ys = G.Y + j * G.ly * G.d;
  if constexpr (WIDE) {
    extern __shared__ double wsm[];
    wide_levels(G, xs, G.lx, ys, G.ly, wsm, lv);
    if (A.norm != SK_NORM_NONE) {
      wide_levels(G, xs, G.lx, xs, G.lx, wsm, dx);
      wide_levels(G, ys, G.ly, ys, G.ly, wsm, dy);
    }
  } else {
    cta_pair_levels(G, xs, G.lx, ys, G.ly, colacc, sm, lv);
    if (A.norm != SK_NORM_NONE) {
      cta_pair_levels(G, xs, G.lx, xs, G.lx, colacc, sm, dx);
      cta_pair_levels(G, ys, G.ly, ys, G.ly, colacc, sm, dy);
    }
  }
  if (threadIdx.x == 0) {
    const double v = finish_entry(lv, M, A.norm, A.norm != SK_NORM_NONE ? dx : nullptr,
                                  A.norm != SK_NORM_NONE ? dy : nullptr);
    A.K[row * A.ldk + j] = v;
    if (sym && j != i) A.K[j * A.ldk + i] = v;
    if (A.levels) {
      for (int m = 0; m <= M; ++m) A.levels[(row * A.ldk + j) * (M + 1) + m] = lv[m];
      if (sym && j != i)
        for (int m = 0; m <= M; ++m) A.levels[(j * A.ldk + i) * (M + 1) + m] = lv[m];
    }
  }
  __syncthreads();
}

// Wide short pairs in batches: the CTA forms WB pairs' matrices one after the
// other (the block DGEMM above), each double-differenced into its slot of the
// CTA's global ring (L2-resident, WP x WP doubles), then WB warps run the
// recursions concurrently — one warp's recursion is a ~100 us latency chain,
// which a lone warp left the other seven waiting on.
constexpr int WB = 8;
constexpr int64_t WSLOT = (int64_t)WP * WP;

// All threads: the matrix of one pair (T1 x T2 increments' kernel values, row
// stride WP, zero beyond T2) into `out`.
__device__ __noinline__ void wide_stage_pair(const Geo &G, const double *xs, int64_t lx,
                                             const double *ys, int64_t ly, double *smem,
                                             double *out) {
  const int T1 = (int)(G.difference ? lx - 1 : lx), T2 = (int)(G.difference ? ly - 1 : ly);
  if (G.M == 0 || T1 <= 0 || T2 <= 0) return;
  wide_point_matrix(G, xs, lx, ys, ly, smem);
  const double *Am = smem;
  const bool diff = G.difference;
  const double sc = wide_dd_scale(G);
  for (int e = threadIdx.x; e < T1 * WP; e += RT) {
    const int i = e / WP, c = e % WP;
    double v = 0.0;
    if (c < T2)
      v = diff ? sc * (Am[(i + 1) * WPS + c + 1] - Am[i * WPS + c + 1] - Am[(i + 1) * WPS + c] +
                       Am[i * WPS + c])
               : Am[i * WPS + c];
    out[e] = v;
  }
  __syncthreads();  // Am is the next pair's
}

// The scan's listed entries (n of them): P = 1 pair per entry, or 3 (the pair
// and both self pairs) when normalised.
template <int MB>
__device__ void redo_wide_batched(const CertArgs &A, int64_t n, double *slots, double *smem,
                                  double (*lvw)[GEN_MAX_LEVELS + 1]) {
  const Geo &G = A.G;
  const int M = G.M, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool sym = A.symmetric, norm = A.norm != SK_NORM_NONE;
  const int P = norm ? 3 : 1, EB = WB / P;
  const auto pair_of = [&](int64_t ee, int role, const double *&p1, int64_t &l1,
                           const double *&p2, int64_t &l2) {
    const int64_t r = ee / G.ny, j = ee % G.ny, i = A.row_begin + r;
    const double *xs = G.X + i * G.lx * G.d, *ys = G.Y + j * G.ly * G.d;
    p1 = role == 2 ? ys : xs;
    l1 = role == 2 ? G.ly : G.lx;
    p2 = role == 1 ? xs : ys;
    l2 = role == 1 ? G.lx : G.ly;
  };
  for (int64_t base = (int64_t)blockIdx.x * EB; base < n; base += (int64_t)gridDim.x * EB) {
    const int nb = (int)(n - base < EB ? n - base : EB);
    for (int b = 0; b < nb * P; ++b) {
      const double *p1, *p2;
      int64_t l1, l2;
      pair_of((int64_t)A.work[1 + base + b / P], b % P, p1, l1, p2, l2);
      wide_stage_pair(G, p1, l1, p2, l2, smem, slots + b * WSLOT);
    }
    if (warp < nb * P) {
      const double *p1, *p2;
      int64_t l1, l2;
      pair_of((int64_t)A.work[1 + base + warp / P], warp % P, p1, l1, p2, l2);
      const int T1 = (int)(G.difference ? l1 - 1 : l1), T2 = (int)(G.difference ? l2 - 1 : l2);
      const double *Ag = slots + warp * WSLOT;
      if (M == 0 || T1 <= 0 || T2 <= 0) {
        if (lane == 0) {
          lvw[warp][0] = 1.0;
          for (int m = 1; m <= M; ++m) lvw[warp][m] = 0.0;
        }
      } else {
        warp_levels<MB>([&](int i, int c) { return Ag[i * WP + c]; }, T1, T2, M, lane, lvw[warp]);
      }
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      const int64_t ee = (int64_t)A.work[1 + base + threadIdx.x];
      const int64_t r = ee / G.ny, j = ee % G.ny, i = A.row_begin + r;
      const int64_t row = sym ? i : r;
      const double *lv = lvw[threadIdx.x * P];
      const double v = finish_entry(lv, M, A.norm, norm ? lvw[threadIdx.x * P + 1] : nullptr,
                                    norm ? lvw[threadIdx.x * P + 2] : nullptr);
      A.K[row * A.ldk + j] = v;
      if (sym && j != i) A.K[j * A.ldk + i] = v;
      if (A.levels) {
        for (int m = 0; m <= M; ++m) A.levels[(row * A.ldk + j) * (M + 1) + m] = lv[m];
        if (sym && j != i)
          for (int m = 0; m <= M; ++m) A.levels[(j * A.ldk + i) * (M + 1) + m] = lv[m];
      }
    }
    __syncthreads();
  }
}

template <bool WIDE>
__global__ void __launch_bounds__(RT, WIDE ? 1 : 2) cert_redo_kernel(CertArgs A) {
  __shared__ double sm[NW * (VMAX + 1) + NW + 3 * (GEN_MAX_LEVELS + 1)];
  __shared__ int64_t list[RT];
  __shared__ int cnt;
  double *lv = sm + NW * (VMAX + 1) + NW, *dx = lv + GEN_MAX_LEVELS + 1, *dy = dx + GEN_MAX_LEVELS + 1;
  const Geo &G = A.G;
  const bool sym = A.symmetric;
  double *colacc = A.scratch + blockIdx.x * A.slot;
  const int64_t n = A.work ? (int64_t)*A.work : A.cap + 1;
  if (WIDE && n <= A.cap) {
    extern __shared__ double wsm[];
    __shared__ double lvw[WB][GEN_MAX_LEVELS + 1];
    if (G.M <= 4)
      redo_wide_batched<4>(A, n, colacc, wsm, lvw);
    else if (G.M <= 8)
      redo_wide_batched<8>(A, n, colacc, wsm, lvw);
    else
      redo_wide_batched<16>(A, n, colacc, wsm, lvw);
    return;
  }
  if (n <= A.cap) {
    for (int64_t q = blockIdx.x; q < n; q += gridDim.x)
      redo_entry<WIDE>(A, (int64_t)A.work[1 + q], colacc, sm, lv, dx, dy);
    return;
  }
  const int64_t total = A.rows * G.ny;
  for (int64_t e0 = (int64_t)blockIdx.x * RT; e0 < total; e0 += (int64_t)gridDim.x * RT) {
    if (threadIdx.x == 0) cnt = 0;
    __syncthreads();
    const int64_t e = e0 + threadIdx.x;
    if (e < total) {
      const int64_t r = e / G.ny, j = e % G.ny, i = A.row_begin + r;
      const int64_t row = sym ? i : r;
      if (!(sym && j < i) && isnan(A.K[row * A.ldk + j])) list[atomicAdd(&cnt, 1)] = e;
    }
    __syncthreads();
    const int nl = cnt;
    __syncthreads();  // every thread has read cnt before it is reset
    for (int q = 0; q < nl; ++q) redo_entry<WIDE>(A, list[q], colacc, sm, lv, dx, dy);
  }
}

// Self levels: level 1 -> exact; noisy, negative or non-finite -> float64.
__global__ void __launch_bounds__(RT, 2) self_cert_kernel(Geo G, double *out, double *scratch,
                                                       int64_t slot) {
  __shared__ double sm[NW * (VMAX + 1) + NW + (GEN_MAX_LEVELS + 1)];
  __shared__ int redo;
  double *lv = sm + NW * (VMAX + 1) + NW;
  const int M = G.M;
  double *colacc = scratch + blockIdx.x * slot;
  for (int64_t i = blockIdx.x; i < G.nx; i += gridDim.x) {
    double *o = out + i * (M + 1);
    const double *x = G.X + i * G.lx * G.d;
    if (threadIdx.x == 0) {
      bool bad = false;
      for (int m = 1; m <= M; ++m) bad |= !(o[m] >= 0.0) || isinf(o[m]);
      if (!bad && G.difference && M >= 1) {
        const double k1e = exact_level1(G.S, x, G.lx, x, G.lx, (int)G.d);
        if (fabs(o[1] - k1e) > CERT_NOISE * fabs(k1e))
          bad = true;
        else
          o[1] = k1e;
      }
      redo = bad;
    }
    __syncthreads();
    if (redo) {
      cta_pair_levels(G, x, G.lx, x, G.lx, colacc, sm, lv);
      if (threadIdx.x == 0)
        for (int m = 0; m <= M; ++m) o[m] = lv[m];
    }
    __syncthreads();
  }
}

Geo geo(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
        int64_t d, const sk_kernel_config &c) {
  Geo G;
  G.X = X;
  G.Y = Y;
  G.nx = nx;
  G.lx = lx;
  G.ny = ny;
  G.ly = ly;
  G.d = d;
  G.S = to_static(c.static_spec);
  G.M = c.n_levels;
  G.difference = c.difference;
  return G;
}

// --- order 1, T' <= 256, d <= WIDE_D: one warp per pair ---------------------
// The row scan above spends a block-wide scan (two barriers) per row on one
// pair; here a warp owns the pair, lanes own C consecutive columns, and a row
// costs the lanes' own point-kernel values (the previous row's kept in
// registers, the column left of a lane's first one by shuffle), one warp scan
// of the M-1 column-accumulator prefixes and the recursion — every state in
// registers, the reference's arithmetic (kernels.py:144-201, :281).
constexpr int WG_WARPS = 8;

template <int C, int MB>
__global__ void __launch_bounds__(32 * WG_WARPS) warp_gram_kernel(GramArgs A) {
  const Geo &G = A.G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, M = G.M, d = (int)G.d;
  const bool diff = G.difference;
  constexpr int VB = MB - 1;
  const int64_t npairs = A.mode == 2 ? G.nx : A.rows * G.ny;
  for (int64_t g = (int64_t)blockIdx.x * WG_WARPS + warp; g < npairs;
       g += (int64_t)gridDim.x * WG_WARPS) {
    int64_t i, j;
    if (A.mode == 2) {
      i = j = g;
    } else {
      i = A.row_begin + g / G.ny;
      j = g % G.ny;
      if (A.mode == 1 && j < i) continue;  // warp-uniform
    }
    const int64_t lxx = G.lx, lyy = A.mode == 2 ? G.lx : G.ly;
    const double *xs = G.X + i * G.lx * d;
    const double *ys = (A.mode == 2 ? G.X : G.Y) + j * lyy * d;
    const int T1 = (int)(diff ? lxx - 1 : lxx), T2 = (int)(diff ? lyy - 1 : lyy);
    double lsum[MB];
#pragma unroll
    for (int m = 0; m < MB; ++m) lsum[m] = 0.0;
    if (M > 0 && T1 > 0 && T2 > 0) {
      const int c0 = lane * C;  // own cells: columns c0 .. c0 + C - 1 of the increment grid
      double ca[VB > 0 ? VB : 1][C];
#pragma unroll
      for (int m = 0; m < VB; ++m)
#pragma unroll
        for (int q = 0; q < C; ++q) ca[m][q] = 0.0;
      // difference: point kernel G(r, c) at the own node columns c0+1 .. c0+C
      // (gp: row r-1) and at column c0 (gl: from the left lane / lane 0 itself)
      double gp[C], gpl = 0.0, yyc[C];
      const bool inner = G.S.kind == SK_LINEAR || G.S.kind == SK_POLYNOMIAL;
#pragma unroll
      for (int q = 0; q < C; ++q) {
        yyc[q] = 0.0;
        if (diff && !inner && c0 + q < T2) {
          const double *yc = ys + (c0 + q + 1) * d;
          for (int k = 0; k < d; ++k) yyc[q] = fma(yc[k], yc[k], yyc[q]);
        }
      }
      if (diff) {
#pragma unroll
        for (int q = 0; q < C; ++q)
          gp[q] = c0 + q < T2 ? static_eval_f64(G.S, xs, ys + (c0 + q + 1) * d, d) : 0.0;
        const double up = __shfl_up_sync(0xffffffffu, gp[C - 1], 1);
        gpl = lane == 0 ? static_eval_f64(G.S, xs, ys, d) : up;
      }
      for (int r = 0; r < T1; ++r) {
        double a[C];
        if (diff) {
          const double *xr = xs + (r + 1) * d;
          double gc[C];
          // the row's |x|^2 once, the columns' |y|^2 from the pair start: each
          // cell is then one dot product (static_eval_f64's arithmetic)
          double xx = 0.0;
          if (!inner)
            for (int k = 0; k < d; ++k) xx = fma(xr[k], xr[k], xx);
#pragma unroll
          for (int q = 0; q < C; ++q) {
            if (c0 + q < T2) {
              const double *yc = ys + (c0 + q + 1) * d;
              double xy = 0.0;
              for (int k = 0; k < d; ++k) xy = fma(xr[k], yc[k], xy);
              gc[q] = inner ? static_from_inner(G.S, xy) : static_from_sq(G.S, xx + yyc[q] - 2.0 * xy);
            } else {
              gc[q] = 0.0;
            }
          }
          const double up = __shfl_up_sync(0xffffffffu, gc[C - 1], 1);
          const double gcl = lane == 0 ? static_eval_f64(G.S, xr, ys, d) : up;
          // kernels.py:281: G[1:,1:] - G[:-1,1:] - G[1:,:-1] + G[:-1,:-1]
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const double g10 = q == 0 ? gcl : gc[q - 1], g00 = q == 0 ? gpl : gp[q - 1];
            a[q] = c0 + q < T2 ? gc[q] - gp[q] - g10 + g00 : 0.0;
          }
#pragma unroll
          for (int q = 0; q < C; ++q) gp[q] = gc[q];
          gpl = gcl;
        } else {
#pragma unroll
          for (int q = 0; q < C; ++q)
            a[q] = c0 + q < T2 ? static_eval_f64(G.S, xs + r * d, ys + (c0 + q) * d, d) : 0.0;
        }
        // exclusive prefix over columns of the column accumulators (old values)
        double pre[VB > 0 ? VB : 1];
#pragma unroll
        for (int m = 0; m < VB; ++m) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < C; ++q) t += ca[m][q];
          pre[m] = t;
        }
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
        for (int q = 0; q < C; ++q) {
          double Rprev = a[q];  // R_1 (0 beyond the own cells)
          lsum[0] += Rprev;
#pragma unroll
          for (int m = 1; m < MB; ++m) {
            if (m < M) {
              const double Rn = a[q] * pre[m - 1];  // R_{m+1} = A * S_m
              lsum[m] += Rn;
              pre[m - 1] += ca[m - 1][q];
              ca[m - 1][q] += Rprev;
              Rprev = Rn;
            }
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
      double lv[MB + 1];
      lv[0] = 1.0;
#pragma unroll
      for (int m = 0; m < MB; ++m) lv[m + 1] = m < M ? lsum[m] : 0.0;
      if (A.mode == 2) {
        for (int m = 0; m <= M; ++m) A.self_out[i * (M + 1) + m] = lv[m];
      } else {
        const bool sym = A.mode == 1;
        const int64_t row = sym ? i : i - A.row_begin;
        if (A.levels) {
          for (int m = 0; m <= M; ++m) A.levels[(row * A.ldk + j) * (M + 1) + m] = lv[m];
          if (sym && j != i)
            for (int m = 0; m <= M; ++m) A.levels[(j * A.ldk + i) * (M + 1) + m] = lv[m];
        }
        if (A.K) {
          const double v = finish_entry(lv, M, A.norm, A.diag_x ? A.diag_x + i * (M + 1) : nullptr,
                                        A.diag_y ? A.diag_y + j * (M + 1) : nullptr);
          A.K[row * A.ldk + j] = v;
          if (sym && j != i) A.K[j * A.ldk + i] = v;
        }
      }
    }
  }
}

bool warp_ok(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  const int p = std::max(1, std::min(c.order, std::max(c.n_levels, 1)));
  const int64_t T = c.difference ? std::max(lx, ly) - 1 : std::max(lx, ly);
  return p == 1 && c.n_levels >= 1 && c.n_levels <= 8 && d <= WIDE_D && T <= 256;
}

int64_t slot_doubles(int64_t lx, int64_t ly, const sk_kernel_config &c) {
  const int64_t L = std::max(lx, ly);
  const int64_t T = c.difference ? std::max<int64_t>(L - 1, 1) : std::max<int64_t>(L, 1);
  // the row buffer of the wide (d > WIDE_D) point-kernel evaluation, then the
  // column accumulators of the long-row (more than 2 columns per thread) variant
  return L + 2 + std::max(c.n_levels - 1, 1) * T;
}

// the certification redo's per-CTA slot: wide short pairs stage WB matrices
int64_t redo_slot_doubles(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  const int64_t slot = slot_doubles(lx, ly, c);
  return wide_short(lx, ly, d, c) ? std::max(slot, WB * WSLOT) : slot;
}

// dynamic shared memory of a row-scan launch: the y staging area, grown to
// hold the column state of long rows (more than 2 columns per thread) too
size_t long_row_smem(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  const int64_t L = std::max(lx, ly), T = c.difference ? L - 1 : L;
  const int64_t NV = std::max(c.n_levels - 1, 0), C = (T + RT - 1) / RT;
  if (d > WIDE_D || L * d > YSTAGE_BYTES / 8 || C <= 2) return YSTAGE_BYTES;
  const size_t need = (size_t)((((L * d + 1) & ~1ll) + NV * C * RT) * 8);
  return need <= (size_t)DYN_SMEM_MAX ? std::max<size_t>(YSTAGE_BYTES, need) : YSTAGE_BYTES;
}

int64_t grid_for(int64_t work, int64_t slot) {
  // enough CTAs to fill the machine, scratch within 256 MiB
  const int64_t cap = std::max<int64_t>(1, (256ll << 20) / (slot * 8));
  return std::max<int64_t>(1, std::min<int64_t>({work, (int64_t)sm_count() * 4, cap}));
}

}  // namespace rowscan

bool warp_gram_ok(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  return rowscan::warp_ok(lx, ly, d, c);
}

bool rowscan_supported(int64_t lx, int64_t ly, const sk_kernel_config &c) {
  const int64_t L = std::max(lx, ly);
  const int64_t T = c.difference ? L - 1 : L;
  const int p = std::max(1, std::min(c.order, std::max(c.n_levels, 1)));
  return p == 1 && c.n_levels <= GEN_MAX_LEVELS && T <= (int64_t)rowscan::RT * rowscan::CMAX;
}

size_t rowscan_workspace_bytes(int64_t npairs, int64_t lx, int64_t ly, const sk_kernel_config &c) {
  using namespace rowscan;
  const int64_t slot = slot_doubles(lx, ly, c);
  return (size_t)grid_for(std::max<int64_t>(npairs, 1), slot) * slot * 8;
}

int rowscan_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                 int64_t ly, int64_t d, int mode, const sk_kernel_config &c, int64_t row_begin,
                 int64_t row_end, const double *diag_x, const double *diag_y, double *K,
                 int64_t ldk, double *levels, double *self_out, void *ws, size_t ws_bytes,
                 cudaStream_t st) {
  using namespace rowscan;
  GramArgs A{};
  A.G = geo(X, nx, lx, Y, ny, ly, d, c);
  A.mode = mode;
  A.row_begin = row_begin;
  A.rows = row_end - row_begin;
  A.norm = c.normalization;
  A.diag_x = diag_x;
  A.diag_y = diag_y;
  A.K = K;
  A.ldk = ldk;
  A.levels = levels;
  A.self_out = self_out;
  const int64_t npairs = mode == 2 ? nx : A.rows * ny;
  if (npairs <= 0) return SK_OK;
  A.slot = slot_doubles(lx, mode == 2 ? lx : ly, c);
  if (warp_ok(lx, mode == 2 ? lx : ly, d, c)) {  // one warp per pair
    const int64_t T = c.difference ? std::max(lx, mode == 2 ? lx : ly) - 1
                                   : std::max(lx, mode == 2 ? lx : ly);
    const int cc = T <= 32 ? 1 : (T <= 64 ? 2 : (T <= 128 ? 4 : 8));
    const unsigned grid = (unsigned)std::min<int64_t>((npairs + WG_WARPS - 1) / WG_WARPS,
                                                      (int64_t)sm_count() * 16);
#define SK_WG(CC, MM) \
    if (cc == CC && (MM == 4 ? c.n_levels <= 4 : c.n_levels > 4)) { \
      warp_gram_kernel<CC, MM><<<grid, 32 * WG_WARPS, 0, st>>>(A); SK_CHECK_LAUNCH(); return SK_OK; }
    SK_WG(1, 4) SK_WG(2, 4) SK_WG(4, 4) SK_WG(8, 4) SK_WG(1, 8) SK_WG(2, 8) SK_WG(4, 8) SK_WG(8, 8)
#undef SK_WG
  }
  if (wide_short(lx, mode == 2 ? lx : ly, d, c)) {  // block DGEMM + one-warp DP per pair
    const int64_t grid = std::min<int64_t>(npairs, (int64_t)sm_count());
    SK_CHECK_CUDA(cudaFuncSetAttribute(gram_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WIDE_SMEM));
    gram_kernel<true><<<(unsigned)grid, RT, WIDE_SMEM, st>>>(A);
    SK_CHECK_LAUNCH();
    return SK_OK;
  }
  const int64_t grid = grid_for(npairs, A.slot);
  if (!ws || ws_bytes < (size_t)(grid * A.slot * 8))
    return fail(SK_ERR_WORKSPACE, "workspace too small for the float64 row-scan kernel");
  A.scratch = (double *)ws;
  const size_t dyn = long_row_smem(lx, mode == 2 ? lx : ly, d, c);
  SK_CHECK_CUDA(cudaFuncSetAttribute(gram_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  gram_kernel<false><<<(unsigned)grid, RT, dyn, st>>>(A);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

// the scan's compacted list: a count and up to min(nx * ny, 4 Mi) entry indices
static int64_t work_list_cap(int64_t nx, int64_t ny) {
  return std::max<int64_t>(1, std::min<int64_t>(nx * ny, 1ll << 22));
}
static size_t work_list_bytes(int64_t nx, int64_t ny) {
  return ((size_t)(work_list_cap(nx, ny) + 1) * 8 + 255) & ~(size_t)255;
}

size_t cert_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                            const sk_kernel_config &c) {
  using namespace rowscan;
  const int64_t slot = redo_slot_doubles(lx, ly, d, c);
  const size_t redo = (size_t)grid_for(1ll << 40, slot) * slot * 8;
  const size_t corners = (size_t)(nx + ny) * 2 * d * 8;  // scan pass, before the redo
  return ((std::max(redo, corners) + 255) & ~(size_t)255) + work_list_bytes(nx, ny);
}

int cert_fixup(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
               int64_t d, int symmetric, const sk_kernel_config &c, int64_t row_begin,
               int64_t row_end, const double *diag_x, const double *diag_y, const float *k1buf,
               double *K, int64_t ldk, double *levels, void *ws, size_t ws_bytes,
               cudaStream_t st) {
  using namespace rowscan;
  CertArgs A{};
  A.G = geo(X, nx, lx, Y, ny, ly, d, c);
  A.symmetric = symmetric;
  A.row_begin = row_begin;
  A.rows = row_end - row_begin;
  A.norm = c.normalization;
  A.diag_x = diag_x;
  A.diag_y = diag_y;
  A.k1buf = reinterpret_cast<const float2 *>(k1buf);
  A.K = K;
  A.ldk = ldk;
  A.levels = levels;
  const int64_t total = A.rows * ny;
  if (total <= 0) return SK_OK;
  if (!ws || ws_bytes < cert_workspace_bytes(nx, lx, ny, ly, d, c))
    return fail(SK_ERR_WORKSPACE, "workspace too small for the certification fix-up");
  A.l1check = c.difference && c.n_levels >= 1;
  {
    // the list lives after the scan / redo scratch
    const int64_t slot = redo_slot_doubles(lx, ly, d, c);
    const size_t redo = (size_t)grid_for(1ll << 40, slot) * slot * 8;
    const size_t corners = (size_t)(nx + ny) * 2 * d * 8;
    A.work = (unsigned long long *)((char *)ws + ((std::max(redo, corners) + 255) & ~(size_t)255));
    A.cap = work_list_cap(nx, ny);
    if (k1buf)
      SK_CHECK_CUDA(cudaMemsetAsync(A.work, 0, 8, st));
    else
      A.work = nullptr;  // no scan: the redo finds the NaN entries itself
  }
  if (k1buf) {
    // transposed corner points of both roles (scan pass only; the redo reuses the space)
    double *Xc = (double *)ws, *Yc = Xc + nx * 2 * d;
    const int64_t tx = nx * 2 * d, ty = ny * 2 * d;
    corners_kernel<<<(unsigned)std::min<int64_t>((tx + 255) / 256, sm_count() * 8), 256, 0, st>>>(
        X, nx, lx, d, Xc);
    SK_CHECK_LAUNCH();
    if (symmetric) {
      Yc = Xc;  // K(X): both roles are X
    } else {
      corners_kernel<<<(unsigned)std::min<int64_t>((ty + 255) / 256, sm_count() * 8), 256, 0, st>>>(
          Y, ny, ly, d, Yc);
      SK_CHECK_LAUNCH();
    }
    const int64_t tiles = ((A.rows + SR - 1) / SR) * ((ny + RT - 1) / RT);
    const unsigned g = (unsigned)std::min<int64_t>(tiles, (int64_t)sm_count() * 8);
    const int k = c.static_spec.kind;
    if (k == SK_LINEAR || k == SK_POLYNOMIAL)
      cert_scan_kernel<true><<<g, RT, 0, st>>>(A, Xc, Yc);
    else
      cert_scan_kernel<false><<<g, RT, 0, st>>>(A, Xc, Yc);
    SK_CHECK_LAUNCH();
  }
  A.slot = redo_slot_doubles(lx, ly, d, c);
  A.scratch = (double *)ws;
  if (wide_short(lx, ly, d, c)) {  // block DGEMM + one-warp DP, one CTA per SM
    const int64_t grid = std::min<int64_t>(sm_count(), (total + RT - 1) / RT);
    SK_CHECK_CUDA(cudaFuncSetAttribute(cert_redo_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)WIDE_SMEM));
    cert_redo_kernel<true><<<(unsigned)grid, RT, WIDE_SMEM, st>>>(A);
  } else {
    const int64_t grid = std::min<int64_t>(grid_for(1ll << 40, A.slot), (total + RT - 1) / RT);
    SK_CHECK_CUDA(cudaFuncSetAttribute(cert_redo_kernel<false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)long_row_smem(lx, ly, d, c)));
    cert_redo_kernel<false><<<(unsigned)grid, RT, long_row_smem(lx, ly, d, c), st>>>(A);
  }
  SK_CHECK_LAUNCH();
  return SK_OK;
}

int cert_self_fixup(const double *X, int64_t n, int64_t l, int64_t d, const sk_kernel_config &c,
                    double *out, void *ws, size_t ws_bytes, cudaStream_t st) {
  using namespace rowscan;
  if (n <= 0) return SK_OK;
  const Geo G = geo(X, n, l, X, n, l, d, c);
  const int64_t slot = slot_doubles(l, l, c);
  const int64_t grid = grid_for(n, slot);
  if (!ws || ws_bytes < (size_t)(grid * slot * 8))
    return fail(SK_ERR_WORKSPACE, "workspace too small for the self-level fix-up");
  const size_t dyn = long_row_smem(l, l, d, c);
  SK_CHECK_CUDA(cudaFuncSetAttribute(self_cert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  self_cert_kernel<<<(unsigned)grid, RT, dyn, st>>>(G, out, (double *)ws, slot);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

}  // namespace sk
