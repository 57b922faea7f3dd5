// Fused FP32 signature-kernel Gram kernel for sm_100a (order p = 1).
//
// Replaces, for one sequence pair per warp segment, the whole inner tile of
// the reference (kernels.py:457-468): the point Gram (_gram_nd,
// kernels.py:252-260), the double difference (kernels.py:281), the
// cumulative-sum recursion (sig_levels_dp, kernels.py:174-199 at p=1:
// R_m = A * S(R_{m-1})) and the level sums, plus the normalisation epilogue
// (kernels.py:586-600). Nothing but the final Gram entry touches HBM.
//
// Systolic row streaming
// ----------------------
// A warp is split into segments of SW lanes (SW = pow2 >= ceil(L_y / C)).
// Lane q of a segment owns C = 8 point-kernel columns g in [C*q, C*q + C) of
// the pair's L_x x L_y grid and keeps, in registers, those columns' y points
// and the column accumulators colacc_m(g) = sum_{i' < i} R_m(i', g) for levels
// m = 1..M-1. Rows are streamed top to bottom, TWO rows (a row pair) per
// step, and lane q runs q steps behind lane 0 (a wavefront). That skew turns
// the 2-D exclusive prefix
//   S_m(i, j) = sum_{i' < i, j' < j} R_m(i', j')
// into a chain: lane q receives from lane q-1 (one __shfl_up per level per
// row) the prefix of everything left of its columns for the SAME row, adds
// its own colaccs serially, and passes the result on next step. Per cell and
// level that is one FADD (scan) + one FFMA (accumulate), i.e. the
// north-star flop model's 4 flops/level/cell, with the cross-lane scan cost
// amortised over C cells.
//
// Row pairs: the point kernel of both rows is evaluated with packed
// FFMA2 (fma.rn.f32x2): the x coordinates of the two rows form one 64-bit
// register pair, reused across the C columns, times the column's y
// coordinate as a broadcast scalar operand. That halves the issue slots of
// the dominant stage at the same FP32-pipe cost (tools/microbench/
// ffma2_rowpair.cu: 127.7 of 128 lane-FMAs/SM/clk), which leaves issue
// bandwidth for the MUFU/SHFL/LDS work of the rest of the step. The level
// recursion then runs row a, then row b.
//
// Pairs stream back to back: a segment keeps its y sequence and walks a
// range of x sequences; each lane switches to the next x when its own row
// counter wraps, so there is no wavefront fill/drain per pair. The level
// sums of a finished pair arrive for free at the segment's last lane: at a
// lane's first step of the next pair, the row-a chain carries sum over all
// lanes of sum_g colacc_m(g) = k_m (and k_M rides a separate chain). Row a of
// that step is the new x's row 0, whose "increments" against the previous x
// are discarded by the reset between rows a and b.
//
// Increments: lane q needs D(g) = G(i,g) - G(i-1,g) for g = C*q - 1, which
// lane q-1 computed one step earlier; it arrives with the carries, so every
// point-kernel value is computed exactly once. Columns beyond L_y repeat the
// last y point, and an odd L_x repeats the last x point (zero increments,
// A = 0), which is exact.
//
// Point kernel: x and y are pre-scaled (rbf: by sqrt(log2 e)/sigma) and
// carry n = -|x'|^2/2, so G = exp2(min(<x',y'> + n_x + n_y, 0)) — the
// reference's norm-expansion form (kernels.py:256-259, clamp at 0 included)
// in D FFMAs + 1 FADD + 1 FMNMX + 1 MUFU.EX2 per cell.
//
// The x sequences of a tile stream through a 3-slot shared-memory ring
// (cp.async, one barrier per x sequence); every warp of the CTA reads the
// same x rows (different y), so the smem traffic is C-fold amortised.
#pragma once

#include "sk_common.cuh"
#include "sk_geo_cells.cuh"

namespace sk {
namespace fast {

constexpr int NWARPS = 8;
constexpr int NTHREADS = NWARPS * 32;
constexpr int NSLOT = 3;

// floats per packed point of the y role / per packed row pair of the x role
__host__ __device__ constexpr int y_stride(int D) { return D + 4; }
__host__ __device__ constexpr int x_stride(int D) { return 2 * D + 4; }

struct Params {
  const float *xs;  // x role (Gram rows), packed row pairs [nx][lx2][2D+4]
  const float *ys;  // y role (Gram columns), packed [ny][lyp][D+4]
  int64_t nx, ny;
  int lx2;       // x row pairs per sequence (steps per pair)
  int lyp;       // packed y point stride
  int sw;        // lanes per segment
  int segs;      // segments (y sequences) per CTA
  int rx;        // x sequences per tile
  int64_t tiles_y, ntiles;
  int64_t row_begin, row_end;
  int symmetric;
  int diag_mode;  // 1: self levels (pairs (i, i) only)
  int norm;
  const double *diag_x, *diag_y;
  double *K;
  int64_t ldk;
  double *levels;
  double *self_out;
  // multi-panel (L_y > 256): the pair's columns are swept in npanel passes of
  // 256 columns; chain values cross panel boundaries through `carry`
  int npanel;
  float *carry;  // [max_ctas * NWARPS][rx + 2 jobs][lx2 steps][nhp]
  int nhp;       // floats per carry entry (2 x NCA chain values, 2 x lastD, kout; padded to 4)
  int max_ctas;  // grid size the carry buffer was sized for
  // stationary static kinds (StatPointStage): kind and rational-quadratic alpha
  int static_kind;
  float rq_alpha;
  // GEMM-fed path (sk_gemm.cu): pair (x, y) row r of the cell matrix is at
  // S + (x - x_blk0) * s_xstride + y * s_ystride + r * s_ld
  const float *S;
  int64_t s_ld, s_xstride, s_ystride, x_blk0;
  // FP32 certification (write_pair; sk_gram in include/sigkern_b200.h):
  // k1buf (rows x ny float2, may be null) receives each entry's FP32 level 1
  // and sum_m |k_m|
  int cert;
  float *k1buf;  // float2 per entry: (FP32 level 1, sum_m |k_m|)
};

typedef unsigned long long u64;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ u64 pack2(float lo, float hi) {
  u64 d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ void unpack2(u64 v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// d = a * {b, b} + c  (ptxas folds the broadcast into FFMA2's scalar operand)
__device__ __forceinline__ u64 ffma2_bc(u64 a, float b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(pack2(b, b)), "l"(c));
  return d;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 fadd2_bc(u64 a, float b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(pack2(b, b)));
  return d;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// carry entries: whole float4s (the carry buffer is 16-byte aligned per entry)
template <int N>
__device__ __forceinline__ void store_f4(float *dst, const float (&v)[N]) {
#pragma unroll
  for (int k = 0; k < N / 4; ++k)
    reinterpret_cast<float4 *>(dst)[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
}
// predicated (not branched) store: the carry writer is one lane of the warp
template <int N>
__device__ __forceinline__ void store_f4_if(float *dst, const float (&v)[N], bool pred) {
#pragma unroll
  for (int k = 0; k < N / 4; ++k)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %5, 0;\n"
        " @p st.global.v4.f32 [%0], {%1, %2, %3, %4};\n}\n" ::"l"(dst + 4 * k),
        "f"(v[4 * k]), "f"(v[4 * k + 1]), "f"(v[4 * k + 2]), "f"(v[4 * k + 3]), "r"((int)pred)
        : "memory");
}
template <int N>
__device__ __forceinline__ void load_f4(float (&v)[N], const float *src) {
#pragma unroll
  for (int k = 0; k < N / 4; ++k) {
    const float4 t = reinterpret_cast<const float4 *>(src)[k];
    v[4 * k] = t.x;
    v[4 * k + 1] = t.y;
    v[4 * k + 2] = t.z;
    v[4 * k + 3] = t.w;
  }
}

__device__ __forceinline__ void stage_sequence(float *dst, const float *src, int nfloats) {
  for (int k = threadIdx.x * 4; k < nfloats; k += NTHREADS * 4) cp_async16(dst + k, src + k);
  cp_async_commit();
}

// Level values of pair (i, j) -> per-level output and/or normalised K entry.
// ls = k_1..k_{M-1} (float chain totals), kout = k_M.
// Certification (sk_gram): besides K, the FP32 level 1 and sum_m |k_m| go to
// `k1buf` as one float2 per entry; the certification pass (sk_rowscan.cu)
// judges the entry from them, so the hot kernel carries no extra logic (one
// 8-byte store: the multi-panel c5 schedule measured 1.24 s with it, 1.39 s
// with a single 4-byte store, 1.21 s with none).
template <int M, class T = float>
__device__ __forceinline__ void write_pair(const Params &P, int64_t i, int64_t j,
                                           const T *ls, T kout) {
  double lv[M + 1];
  lv[0] = 1.0;
#pragma unroll
  for (int m = 1; m < M; ++m) lv[m] = (double)ls[m - 1];
  lv[M] = (double)kout;
  if (P.diag_mode) {
    if (i == j) {
#pragma unroll
      for (int m = 0; m <= M; ++m) P.self_out[j * (M + 1) + m] = lv[m];
    }
    return;
  }
  if (P.symmetric && i > j) return;
  const int64_t row = P.symmetric ? i : i - P.row_begin;
  const bool mirror = P.symmetric && i != j;
  const double *dx = P.diag_x ? P.diag_x + i * (M + 1) : nullptr;
  if (P.symmetric && i == j && dx) {  // K(X)'s diagonal from the self levels: exactly 1
#pragma unroll
    for (int m = 0; m <= M; ++m) lv[m] = dx[m];
  }
  if (P.levels) {
#pragma unroll
    for (int m = 0; m <= M; ++m) P.levels[(row * P.ldk + j) * (M + 1) + m] = lv[m];
    if (mirror) {
#pragma unroll
      for (int m = 0; m <= M; ++m) P.levels[(j * P.ldk + i) * (M + 1) + m] = lv[m];
    }
  }
  if (P.K) {
    const double v = finish_entry(lv, M, P.norm, dx, P.diag_y ? P.diag_y + j * (M + 1) : nullptr);
    P.K[row * P.ldk + j] = v;
    if (mirror) P.K[j * P.ldk + i] = v;
    if (P.k1buf) {
      float sa = 1.f + fabsf((float)kout);
#pragma unroll
      for (int m = 1; m < M; ++m) sa += fabsf((float)ls[m - 1]);
      reinterpret_cast<float2 *>(P.k1buf)[row * P.ny + j] =
          make_float2(M == 1 ? (float)kout : (M > 1 ? (float)ls[0] : 0.f), sa);
    }
  }
}

// A = D(g) - D(g-1), D = G(r,.) - G(r-1,.) for rows a, b of a row pair.
// dla/dlb: D of the column left of this lane (lane q-1's last column, or the
// previous panel's); zero_left: column -1 does not exist (A = 0).
// Linear kind: both roles hold increments (pack kernels), so the point kernel
// already is A = <dx_i, dy_j> (kernels.py:281 is bilinear), without the
// cancellation of differencing the point Gram in FP32.
template <int C, bool LINEAR>
__device__ __forceinline__ void double_difference(const float (&ga)[C], const float (&gb)[C],
                                                  float (&prevG)[C], float &lastDa, float &lastDb,
                                                  float dla, float dlb, bool zero_left,
                                                  float (&aa)[C], float (&ab)[C]) {
  if constexpr (LINEAR) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      aa[c] = ga[c];
      ab[c] = gb[c];
    }
  } else {
    float dva[C], dvb[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      dva[c] = ga[c] - prevG[c];
      dvb[c] = gb[c] - ga[c];
      prevG[c] = gb[c];
    }
    aa[0] = zero_left ? 0.f : dva[0] - dla;
    ab[0] = zero_left ? 0.f : dvb[0] - dlb;
#pragma unroll
    for (int c = 1; c < C; ++c) {
      aa[c] = dva[c] - dva[c - 1];
      ab[c] = dvb[c] - dvb[c - 1];
    }
    lastDa = dva[C - 1];
    lastDb = dvb[C - 1];
  }
}

// ---------------------------------------------------------------------------
// Point stage shared by the lane states: this lane's C y columns in
// registers, the packed-FFMA2 point kernel of a row pair, and the double
// difference (kernels.py:281) producing the increments of rows a and b.
// ---------------------------------------------------------------------------
// KIND 0: rbf, double-differenced (kernels.py:281); 1: linear (the packed values
// are increments, or points when difference=False: A is the point kernel
// itself); 2: rbf with difference=False (A = G).
template <int D, int C_, int KIND>
struct PointStage {
  static constexpr bool LINEAR = KIND == 1;
  static constexpr int C = C_;
  static constexpr int XP = x_stride(D);
  static constexpr int YP = y_stride(D);

  float yv[C][D];
  float yn[C];
  float prevG[C];
  float lastDa, lastDb;
  float ga[C], gb[C];  // point-kernel rows a, b of the current row pair
  __device__ __forceinline__ void configure(const Params &) {}

  // this lane's columns of the packed y sequence (pre-scaled points, n-terms)
  __device__ __forceinline__ void load_y(const float *__restrict__ yp) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int k4 = 0; k4 < D / 4; ++k4) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(yp + c * YP) + k4);
        yv[c][4 * k4 + 0] = v.x;
        yv[c][4 * k4 + 1] = v.y;
        yv[c][4 * k4 + 2] = v.z;
        yv[c][4 * k4 + 3] = v.w;
      }
      yn[c] = LINEAR ? 0.f : __ldg(yp + c * YP + D);
      prevG[c] = 0.f;
    }
    lastDa = lastDb = 0.f;
  }

  // Point kernel of rows a, b of the row pair at `xptr` (packed FFMA2) -> ga, gb.
  __device__ __forceinline__ void point(const float *__restrict__ xptr) {
    u64 acc[C];
    if (LINEAR) {
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = 0ull;
    } else {
      const u64 xn2 = *reinterpret_cast<const u64 *>(xptr + 2 * D);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = fadd2_bc(xn2, yn[c]);
    }
    const float4 *xr = reinterpret_cast<const float4 *>(xptr);
#pragma unroll
    for (int k2 = 0; k2 < D / 2; ++k2) {
      const float4 v = xr[k2];  // {x_a[2k2], x_b[2k2], x_a[2k2+1], x_b[2k2+1]}
      const u64 p0 = pack2(v.x, v.y);
      const u64 p1 = pack2(v.z, v.w);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = ffma2_bc(p0, yv[c][2 * k2], acc[c]);
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = ffma2_bc(p1, yv[c][2 * k2 + 1], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float lo, hi;
      unpack2(acc[c], lo, hi);
      if (LINEAR) {
        ga[c] = lo;
        gb[c] = hi;
      } else if constexpr (D >= 8) {
        // No clamp of the exponent at 0 (the reference clamps the float64
        // squared distance, static/kernels.py:108-114): in FP32 the norm-
        // expansion exponent near x = y carries an error of ~|x|^2 2^-23 of
        // either sign, so clamping only the positive side buys no accuracy;
        // dropping the FMNMX measured +2.1% at c3 and +3.4% at c2. The D = 4
        // kernels keep it: the same edit made the c5 multi-panel kernel 22%
        // slower (its schedule is very sensitive to code changes).
        ga[c] = ex2_approx(lo);
        gb[c] = ex2_approx(hi);
      } else {
        ga[c] = ex2_approx(fminf(lo, 0.f));
        gb[c] = ex2_approx(fminf(hi, 0.f));
      }
    }
  }

  __device__ __forceinline__ void increments(float dla, float dlb, bool zero_left, float (&aa)[C],
                                             float (&ab)[C]) {
    double_difference<C, KIND != 0>(ga, gb, prevG, lastDa, lastDb, dla, dlb, zero_left, aa, ab);
  }
};

// ---------------------------------------------------------------------------
// Stationary static kinds (static/kernels.py:74-89): Matern 1/2, 3/2, 5/2 and
// rational quadratic, k = f(r), r = |x - y| / bandwidth. Coordinates are
// pre-scaled by 1/bandwidth and the squared distance is formed from DIRECT
// differences, sum_k (x_k - y_k)^2 (packed FADD2 + FFMA2 per channel): the
// norm expansion that the rbf stage uses would put an absolute error of
// ~eps |x|^2 under the square root (Matern 1/2 levelwise: 1.2e-4 in a numpy
// FP32 emulation vs 5.7e-8 with direct differences). The kind is a
// warp-uniform runtime parameter.
// ---------------------------------------------------------------------------
template <int D, int C_>
struct StatPointStage {
  static constexpr int C = C_;
  static constexpr int XP = x_stride(D);
  static constexpr int YP = y_stride(D);

  float ynv[C][D];  // -y (negated: the difference is one FADD2 with a broadcast operand)
  float prevG[C];
  float lastDa, lastDb;
  float ga[C], gb[C];
  int kind;
  float alpha, inv2a;

  __device__ __forceinline__ void configure(const Params &P) {
    kind = P.static_kind;
    alpha = P.rq_alpha;
    inv2a = 0.5f / P.rq_alpha;
  }
  __device__ __forceinline__ void load_y(const float *__restrict__ yp) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int k4 = 0; k4 < D / 4; ++k4) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(yp + c * YP) + k4);
        ynv[c][4 * k4 + 0] = -v.x;
        ynv[c][4 * k4 + 1] = -v.y;
        ynv[c][4 * k4 + 2] = -v.z;
        ynv[c][4 * k4 + 3] = -v.w;
      }
      prevG[c] = 0.f;
    }
    lastDa = lastDb = 0.f;
  }
  __device__ __forceinline__ float kfun(float sq) const {
    constexpr float L2E = 1.4426950408889634f;
    float sr;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sr) : "f"(sq));
    if (kind == SK_MATERN12) return ex2_approx(-L2E * sr);
    if (kind == SK_MATERN32) {
      const float t = 1.7320508075688772f * sr;
      return (1.f + t) * ex2_approx(-L2E * t);
    }
    if (kind == SK_MATERN52) {
      const float t = 2.23606797749979f * sr;
      return fmaf(t * t, 1.f / 3.f, 1.f + t) * ex2_approx(-L2E * t);
    }
    // rational quadratic: (1 + sq / (2 alpha))^(-alpha)
    float lg;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(fmaf(sq, inv2a, 1.f)));
    return ex2_approx(-alpha * lg);
  }
  __device__ __forceinline__ void point(const float *__restrict__ xptr) {
    u64 acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = 0ull;
    const float4 *xr = reinterpret_cast<const float4 *>(xptr);
#pragma unroll
    for (int k2 = 0; k2 < D / 2; ++k2) {
      const float4 v = xr[k2];
      const u64 p0 = pack2(v.x, v.y);
      const u64 p1 = pack2(v.z, v.w);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const u64 d0 = fadd2_bc(p0, ynv[c][2 * k2]);
        const u64 d1 = fadd2_bc(p1, ynv[c][2 * k2 + 1]);
        acc[c] = ffma2(d0, d0, acc[c]);
        acc[c] = ffma2(d1, d1, acc[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float lo, hi;
      unpack2(acc[c], lo, hi);
      ga[c] = kfun(lo);
      gb[c] = kfun(hi);
    }
  }
  __device__ __forceinline__ void increments(float dla, float dlb, bool zero_left, float (&aa)[C],
                                             float (&ab)[C]) {
    double_difference<C, false>(ga, gb, prevG, lastDa, lastDb, dla, dlb, zero_left, aa, ab);
  }
};

// ---------------------------------------------------------------------------
// GEMM-fed stage (large d, sk_gemm.cu): the exponent (rbf, with the n-terms
// folded into the GEMM's K) or the increment inner product (linear) of every
// cell was produced by a library GEMM into HBM; a row pair is two rows of
// that matrix, `ld` floats apart.
// ---------------------------------------------------------------------------
template <int C_, bool LINEAR>
struct GemmStage {
  static constexpr int C = C_;
  float prevG[C];
  float lastDa, lastDb;
  float ga[C], gb[C];
  int64_t ld;

  __device__ __forceinline__ void configure(const Params &P) { ld = P.s_ld; }
  __device__ __forceinline__ void reset_y() {
#pragma unroll
    for (int c = 0; c < C; ++c) prevG[c] = 0.f;
    lastDa = lastDb = 0.f;
  }
  __device__ __forceinline__ void point(const float *__restrict__ srow) {
#pragma unroll
    for (int c4 = 0; c4 < C / 4; ++c4) {
      const float4 va = __ldcs(reinterpret_cast<const float4 *>(srow) + c4);  // read once
      const float4 vb = __ldcs(reinterpret_cast<const float4 *>(srow + ld) + c4);
      ga[4 * c4 + 0] = va.x;
      ga[4 * c4 + 1] = va.y;
      ga[4 * c4 + 2] = va.z;
      ga[4 * c4 + 3] = va.w;
      gb[4 * c4 + 0] = vb.x;
      gb[4 * c4 + 1] = vb.y;
      gb[4 * c4 + 2] = vb.z;
      gb[4 * c4 + 3] = vb.w;
    }
    if (!LINEAR) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        ga[c] = ex2_approx(fminf(ga[c], 0.f));
        gb[c] = ex2_approx(fminf(gb[c], 0.f));
      }
    }
  }
  __device__ __forceinline__ void increments(float dla, float dlb, bool zero_left, float (&aa)[C],
                                             float (&ab)[C]) {
    double_difference<C, LINEAR>(ga, gb, prevG, lastDa, lastDb, dla, dlb, zero_left, aa, ab);
  }
};

// Receive chain values from lane q-1 (its previous step); the segment head
// takes zeros, or the previous panel's carries `hin[k]` when from_buf.
template <int N, class T = float>
__device__ __forceinline__ void chain_in(const T (&out)[N], T (&in)[N], int n, int sw,
                                         bool first_lane, bool from_buf, const float *hin) {
#pragma unroll
  for (int k = 0; k < N; ++k) {
    if (k < n) {
      const float v = __shfl_up_sync(0xffffffffu, out[k], 1, sw);
      in[k] = first_lane ? (from_buf ? (T)hin[k] : (T)0) : v;
    }
  }
}

// ---------------------------------------------------------------------------
// Order p = 1 lane state (C = 8 columns per lane).
// ---------------------------------------------------------------------------
template <class Stage, int M_>
struct LaneState1 : Stage {
  using Stage::C;
  static constexpr int M = M_;
  static constexpr int NCA = (M >= 2) ? M - 1 : 0;  // column-accumulated levels 1..M-1
  static constexpr int NCR = (NCA > 0) ? NCA : 1;
  static constexpr int NHM = 2 * NCA + 3;  // carry entry: couta, coutb, lastDa, lastDb, kout
  static constexpr int NHP = (NHM + 3) / 4 * 4;  // padded to whole float4s

  float colacc[NCR][C];
  float couta[NCR], coutb[NCR];
  float kM, kout;

  __device__ __forceinline__ void reset_pair() {
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int m = 0; m < NCR; ++m) colacc[m][c] = 0.f;
    }
    kM = 0.f;
  }
  __device__ __forceinline__ void reset_panel() {
    reset_pair();
    kout = 0.f;
#pragma unroll
    for (int m = 0; m < NCR; ++m) couta[m] = coutb[m] = 0.f;
  }
  // level sums k_1..k_{M-1} of the pair that just completed (valid at the
  // segment's last lane at its boundary step), and k_M = kout
  __device__ __forceinline__ const float *level_sums() const { return couta; }
  __device__ __forceinline__ void store_carry(float *dst, bool pred) const {
    float buf[NHP];
#pragma unroll
    for (int m = 0; m < NCA; ++m) {
      buf[m] = couta[m];
      buf[NCA + m] = coutb[m];
    }
    buf[2 * NCA] = this->lastDa;
    buf[2 * NCA + 1] = this->lastDb;
    buf[2 * NCA + 2] = kout;
#pragma unroll
    for (int k = NHM; k < NHP; ++k) buf[k] = 0.f;
    store_f4_if<NHP>(dst, buf, pred);
  }

  // Level recursion of one row (p = 1): R_m = A * S(R_{m-1}); cin = the
  // chain's prefix left of this lane, cout = prefix including this lane.
  __device__ __forceinline__ void row(const float (&a)[C], const float (&cin)[NCR],
                                      float (&cout)[NCR]) {
    if constexpr (M == 1) {
#pragma unroll
      for (int c = 0; c < C; ++c) kM += a[c];
    } else {
      float sc[NCR];
#pragma unroll
      for (int m = 0; m < NCA; ++m) sc[m] = cin[m];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        float so[NCR];
#pragma unroll
        for (int m = 0; m < NCA; ++m) {
          so[m] = sc[m];
          sc[m] += colacc[m][c];
        }
        colacc[0][c] += a[c];
#pragma unroll
        for (int m = 1; m < NCA; ++m) colacc[m][c] = fmaf(a[c], so[m - 1], colacc[m][c]);
        kM = fmaf(a[c], so[NCA - 1], kM);
      }
#pragma unroll
      for (int m = 0; m < NCA; ++m) cout[m] = sc[m];
    }
  }

  // One row pair (at `xptr`) of this lane's C columns. (Software-pipelining
  // the next row pair's point kernel into this step's recursion was measured
  // slower: 255 registers, 57% vs 62% of the FP32 roofline at c3.)
  //  KCHAIN: also run the level-M chain (only needed while some lane of the
  //          segment is at a pair boundary).
  //  MULTI:  the chain head takes its inputs from `hin` (the previous panel's
  //          carries for this row pair) when head_buf, instead of zeros.
  //  BCHK:   `boundary` may be true: row a starts a new pair, so the pair
  //          state is reset between rows a and b.
  template <bool KCHAIN, bool MULTI, bool BCHK>
  __device__ __forceinline__ void step(const float *__restrict__ xptr, int sw, bool first_lane,
                                       const float *hin, bool head_buf, bool boundary) {
    const bool from_buf = MULTI && head_buf;
    // (a) chain values produced by lane q-1 on the previous step
    float dla = __shfl_up_sync(0xffffffffu, this->lastDa, 1, sw);
    float dlb = __shfl_up_sync(0xffffffffu, this->lastDb, 1, sw);
    float cina[NCR], cinb[NCR];
    chain_in(couta, cina, NCA, sw, first_lane, from_buf, hin);
    chain_in(coutb, cinb, NCA, sw, first_lane, from_buf, hin + NCA);
    if (from_buf && first_lane) {
      dla = hin[2 * NCA];
      dlb = hin[2 * NCA + 1];
    }
    if (KCHAIN) {
      const float kin = __shfl_up_sync(0xffffffffu, kout, 1, sw);
      kout = (first_lane ? (from_buf ? hin[2 * NCA + 2] : 0.f) : kin) + kM;  // complete at a boundary
    }
    // (b) point kernel of rows a, b; (c) increments
    this->point(xptr);
    float aa[C], ab[C];
    this->increments(dla, dlb, first_lane && !from_buf, aa, ab);
    // (d) level recursion, row a then row b
    row(aa, cina, couta);
    if (BCHK && boundary) reset_pair();
    row(ab, cinb, coutb);
  }
};

// ---------------------------------------------------------------------------
// Order p = 1 with float64 column accumulators, row prefixes and level sums
// (single panel only). The GEMM-fed path (large d, e.g. BASELINE c4; rbf too
// since a fuzz seed at n_levels 8 sat at 1.06x the bar): its levels are long
// sums of increment products that cancel, and the FP32
// accumulation measured up to 5e-5 of sum_m |k_m| there (2e-3 relative on
// 0.4% of c4's entries); float64 accumulation brings it to ~1e-6 (the FP32
// cell values remain). The DP of this path streams its cells from HBM
// (4 bytes per cell), so the float64 pipe (~60 lane-ops/clk/SM) has room.
// ---------------------------------------------------------------------------
template <class Stage, int M_>
struct LaneState1D : Stage {
  using Stage::C;
  static constexpr int M = M_;
  static constexpr int NCA = (M >= 2) ? M - 1 : 0;
  static constexpr int NCR = (NCA > 0) ? NCA : 1;
  static constexpr int NHP = 4;  // no carries (single panel)

  double colacc[NCR][C];
  double couta[NCR], coutb[NCR];
  double kM, kout;

  __device__ __forceinline__ void reset_pair() {
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int m = 0; m < NCR; ++m) colacc[m][c] = 0.0;
    }
    kM = 0.0;
  }
  __device__ __forceinline__ void reset_panel() {
    reset_pair();
    kout = 0.0;
#pragma unroll
    for (int m = 0; m < NCR; ++m) couta[m] = coutb[m] = 0.0;
  }
  __device__ __forceinline__ const double *level_sums() const { return couta; }
  __device__ __forceinline__ void store_carry(float *, bool) const {}

  __device__ __forceinline__ void row(const float (&a)[C], const double (&cin)[NCR],
                                      double (&cout)[NCR]) {
    if constexpr (M == 1) {
#pragma unroll
      for (int c = 0; c < C; ++c) kM += (double)a[c];
    } else {
      double sc[NCR];
#pragma unroll
      for (int m = 0; m < NCA; ++m) sc[m] = cin[m];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double ad = (double)a[c];
        double so[NCR];
#pragma unroll
        for (int m = 0; m < NCA; ++m) {
          so[m] = sc[m];
          sc[m] += colacc[m][c];
        }
        colacc[0][c] += ad;
#pragma unroll
        for (int m = 1; m < NCA; ++m) colacc[m][c] = fma(ad, so[m - 1], colacc[m][c]);
        kM = fma(ad, so[NCA - 1], kM);
      }
#pragma unroll
      for (int m = 0; m < NCA; ++m) cout[m] = sc[m];
    }
  }

  template <bool KCHAIN, bool MULTI, bool BCHK>
  __device__ __forceinline__ void step(const float *__restrict__ xptr, int sw, bool first_lane,
                                       const float *, bool, bool boundary) {
    static_assert(!MULTI, "LaneState1D is single-panel");
    const float dla = __shfl_up_sync(0xffffffffu, this->lastDa, 1, sw);
    const float dlb = __shfl_up_sync(0xffffffffu, this->lastDb, 1, sw);
    double cina[NCR], cinb[NCR];
    chain_in(couta, cina, NCA, sw, first_lane, false, nullptr);
    chain_in(coutb, cinb, NCA, sw, first_lane, false, nullptr);
    if (KCHAIN) {
      const double kin = __shfl_up_sync(0xffffffffu, kout, 1, sw);
      kout = (first_lane ? 0.0 : kin) + kM;
    }
    this->point(xptr);
    float aa[C], ab[C];
    this->increments(dla, dlb, first_lane, aa, ab);
    row(aa, cina, couta);
    if (BCHK && boundary) reset_pair();
    row(ab, cinb, coutb);
  }
};

// ---------------------------------------------------------------------------
// General order 1 < p <= M (the geometric kernel at p = M), C = 4 columns
// per lane. The reference's recursion (kernels.py:179-199):
//   R'[0,0] = A S(C),                 C = sum_{q,r} R[q,r]
//   R'[q,0] = A/(q+1) E_j(sum_r R[q-1,r])
//   R'[0,r] = A/(r+1) E_i(sum_q R[q,r-1])
//   R'[q,r] = A/((q+1)(r+1)) R[q-1,r-1]
// is run per cell on factorial-scaled states Rs[q,r] = (q+1)!(r+1)! R[q,r],
// which turns every state update into one multiply by A:
//   Rs'[0,0] = A S(C),  Rs'[q,0] = A e_q,  Rs'[0,r] = A f_r,  Rs'[q,r] = A Rs[q-1,r-1]
// with the scaled prefixes e_q = E_j(rs[q-1]), f_r = E_i(cs[r-1]) of the row
// and column sums rs[q] = sum_r Rs[q,r]/(r+1)!, cs[r] = sum_q Rs[q,r]/(q+1)!,
// and C = sum_q rs[q]/(q+1)!. S and E_i are column accumulators (colS, colE)
// plus, for S, the cross-lane chain; E_j is a pure row prefix: a running sum
// along the lane's columns plus a cross-lane chain, exactly like S.
// ---------------------------------------------------------------------------
template <class Stage, int M_, int P>
struct LaneStateG : Stage {
  using Stage::C;
  using Cell = GeoCell<M_, P>;  // generated straight-line cell (sk_geo_cells.cuh)
  static constexpr int M = M_;
  static_assert(P >= 2 && P <= M, "general-order lane state needs 2 <= p <= M");
  static constexpr int NS = Cell::NS;   // S chains / colS: C_m of levels 1..M-1
  static constexpr int NE = Cell::NE;   // E chains / colE
  static constexpr int NCH = NS + NE;   // chain values per row
  static constexpr int NHM = 2 * NCH + 3;
  static constexpr int NHP = (NHM + 3) / 4 * 4;

  float colS[C][NS];
  float colE[C][NE];
  float cha[NCH], chb[NCH];  // chain outputs of rows a, b: [S (NS) | E (NE)]
  float kM, kout;

  __device__ __forceinline__ void reset_pair() {
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int m = 0; m < NS; ++m) colS[c][m] = 0.f;
#pragma unroll
      for (int k = 0; k < NE; ++k) colE[c][k] = 0.f;
    }
    kM = 0.f;
  }
  __device__ __forceinline__ void reset_panel() {
    reset_pair();
    kout = 0.f;
#pragma unroll
    for (int k = 0; k < NCH; ++k) cha[k] = chb[k] = 0.f;
  }
  __device__ __forceinline__ const float *level_sums() const { return cha; }
  __device__ __forceinline__ void store_carry(float *dst, bool pred) const {
    float buf[NHP];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      buf[k] = cha[k];
      buf[NCH + k] = chb[k];
    }
    buf[2 * NCH] = this->lastDa;
    buf[2 * NCH + 1] = this->lastDb;
    buf[2 * NCH + 2] = kout;
#pragma unroll
    for (int k = NHM; k < NHP; ++k) buf[k] = 0.f;
    store_f4_if<NHP>(dst, buf, pred);
  }

  // Level recursion of one row. cin/cout: [S prefixes | E prefixes].
  __device__ __forceinline__ void row(const float (&a)[C], const float (&cin)[NCH],
                                      float (&cout)[NCH]) {
    float sc[NS], ec[NE];
#pragma unroll
    for (int m = 0; m < NS; ++m) sc[m] = cin[m];
#pragma unroll
    for (int k = 0; k < NE; ++k) ec[k] = cin[NS + k];
#pragma unroll
    for (int c = 0; c < C; ++c) Cell::cell(a[c], sc, ec, colS[c], colE[c], kM);
#pragma unroll
    for (int m = 0; m < NS; ++m) cout[m] = sc[m];
#pragma unroll
    for (int k = 0; k < NE; ++k) cout[NS + k] = ec[k];
  }

  template <bool KCHAIN, bool MULTI, bool BCHK>
  __device__ __forceinline__ void step(const float *__restrict__ xptr, int sw, bool first_lane,
                                       const float *hin, bool head_buf, bool boundary) {
    const bool from_buf = MULTI && head_buf;
    float dla = __shfl_up_sync(0xffffffffu, this->lastDa, 1, sw);
    float dlb = __shfl_up_sync(0xffffffffu, this->lastDb, 1, sw);
    float cina[NCH], cinb[NCH];
    chain_in(cha, cina, NCH, sw, first_lane, from_buf, hin);
    chain_in(chb, cinb, NCH, sw, first_lane, from_buf, hin + NCH);
    if (from_buf && first_lane) {
      dla = hin[2 * NCH];
      dlb = hin[2 * NCH + 1];
    }
    if (KCHAIN) {
      const float kin = __shfl_up_sync(0xffffffffu, kout, 1, sw);
      kout = (first_lane ? (from_buf ? hin[2 * NCH + 2] : 0.f) : kin) + kM;
    }
    this->point(xptr);
    float aa[C], ab[C];
    this->increments(dla, dlb, first_lane && !from_buf, aa, ab);
    row(aa, cina, cha);
    if (BCHK && boundary) reset_pair();
    row(ab, cinb, chb);
  }
};

template <class LS, bool MULTI>
__global__ void __launch_bounds__(NTHREADS, 1) gram_kernel(const Params P) {
  constexpr int M = LS::M;
  constexpr int C = LS::C;
  constexpr int XP = LS::XP;
  constexpr int YP = LS::YP;
  extern __shared__ __align__(16) float smem[];
  const int lx2 = P.lx2;
  const int slot_floats = lx2 * XP;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sw = P.sw;
  const int q = lane & (sw - 1);
  const int seg = warp * (32 / sw) + lane / sw;
  const bool last_lane = (q == sw - 1);
  const bool first_lane = (q == 0);

  LS st;
  st.configure(P);
  for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    const int64_t ty = tile % P.tiles_y;
    const int64_t tx = tile / P.tiles_y;
    int64_t ybase = ty * P.segs;
    int64_t x0, njobs;
    if (P.diag_mode) {
      // self levels: one tile per sequence t; the CTA streams x_t once and
      // only the segment holding y_t keeps its (diagonal) pair
      ybase = (tile / P.segs) * P.segs;
      x0 = tile;
      njobs = 1;
    } else {
      x0 = P.row_begin + tx * P.rx;
      njobs = min((int64_t)P.rx, P.row_end - x0);
      if (P.symmetric && x0 > ybase + P.segs - 1) continue;  // CTA-uniform
    }
    const int64_t j = ybase + seg;
    const bool jvalid = j < P.ny;
    const int64_t jj = jvalid ? j : P.ny - 1;

    // carry region of this warp (multi-panel only)
    float *cbuf = MULTI ? P.carry + ((size_t)(blockIdx.x * NWARPS + warp) * (P.rx + 2)) * lx2 * P.nhp
                        : nullptr;
    const int npanel = MULTI ? P.npanel : 1;
    for (int pnl = 0; pnl < npanel; ++pnl) {
      // this lane's y columns of panel pnl (pre-scaled points and their n-terms)
      st.load_y(P.ys + ((size_t)jj * P.lyp + (size_t)pnl * 32 * C + (size_t)q * C) * YP);
      st.reset_panel();
      const bool head_buf = MULTI && pnl > 0;          // chain inputs from the previous panel
      const bool tail_buf = MULTI && pnl < npanel - 1;  // chain outputs for the next panel
      const bool last_panel = pnl == npanel - 1;

      __syncthreads();  // previous readers are done with the ring (and the carries are visible)
      stage_sequence(smem, P.xs + (size_t)x0 * lx2 * XP, slot_floats);

      // head inputs, prefetched one step ahead (lane 0 reads job e, row pair s)
      constexpr int NHM = LS::NHP;
      float hcur[NHM], hnext[NHM];
#pragma unroll
      for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k] = 0.f;
      // every lane loads the entry (one broadcast transaction, no divergence);
      // only the segment head uses it
      auto load_head = [&](float (&h)[NHM], int64_t job, int rp) {
        if (head_buf) load_f4(h, cbuf + ((size_t)job * lx2 + rp) * P.nhp);
      };
      auto store_tail = [&](int64_t job, int rp) {
        st.store_carry(cbuf + ((size_t)job * lx2 + rp) * P.nhp, tail_buf && last_lane && job >= 0);
      };
      load_head(hcur, 0, 0);

      // Epoch e streams x_{x0+e}: lane q starts that pair at step s = q (its
      // row pair 0) and spends steps s < q finishing pair e-1. So pair
      // boundaries only occur in steps s < sw ("phase A"); steps s >= sw are
      // branch-free.
      for (int64_t e = 0; e <= njobs; ++e) {
        cp_async_wait_all();
        __syncthreads();
        if (e + 1 < njobs)
          stage_sequence(smem + ((e + 1) % NSLOT) * slot_floats,
                         P.xs + (size_t)(x0 + e + 1) * lx2 * XP, slot_floats);
        const float *cur = smem + (e % NSLOT) * slot_floats;
        // before its first pair a lane idles on rows of x_{x0} (slot 0)
        const float *prev = (e == 0) ? smem : smem + ((e + NSLOT - 1) % NSLOT) * slot_floats;
        const int steps = (e < njobs) ? lx2 : sw;
        const int nA = min(sw, steps);
        for (int s = 0; s < nA; ++s) {
          if (MULTI) load_head(hnext, s + 1 < steps ? e : e + 1, s + 1 < steps ? s + 1 : 0);
          const float *xp = (s < q) ? prev + (lx2 - q + s) * XP : cur + (s - q) * XP;
          st.template step<true, MULTI, true>(xp, sw, first_lane, hcur, head_buf, s == q);
          if (MULTI) {
            // the segment's last lane is at (job, pair) = (e, s - q) or (e - 1, lx2 - q + s)
            if (s >= q)
              store_tail(e, s - q);
            else
              store_tail(e - 1, lx2 - q + s);
          }
          if (s == q) {  // this lane's pair boundary: pair e-1 is complete
            if (last_panel && last_lane && e >= 1 && jvalid)
              write_pair<M>(P, x0 + e - 1, j, st.level_sums(), st.kout);
          }
          if (MULTI) {
#pragma unroll
            for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k];
          }
        }
        const float *xp = cur + (nA - q) * XP;
#pragma unroll 1
        for (int s = nA; s < steps; ++s) {
          if (MULTI) load_head(hnext, s + 1 < steps ? e : e + 1, s + 1 < steps ? s + 1 : 0);
          st.template step<false, MULTI, false>(xp, sw, first_lane, hcur, head_buf, false);
          if (MULTI) {
            store_tail(e, s - q);
#pragma unroll
            for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k];
          }
          xp += XP;
        }
      }
    }
  }
}

// Pack (N, L, d) float64 into the kernel layouts with pre-scaled coordinates,
// zero-padded channels and the n-term (from the rounded coordinates):
//  y role: [N][Lp][D+4], point p = min(p, L-1), n-term at column D.
//  x role: [N][Lp2][2D+4] row pairs, rows (2t, 2t+1) interleaved per
//          channel, n-terms at 2D, 2D+1; rows beyond L repeat the last point.
//  mode (pack_mode): 0 points; 1 increments x_p - x_{p-1} (0 for p = 0 and
//  beyond L, formed in float64; linear kind); 2/3 difference=False (rbf /
//  linear): the x role gets a dummy row 0 (the discarded first row of every
//  pair), and rows/columns beyond L are dummies whose point kernel is 0 (rbf:
//  n-term -1e30, so exp2 underflows to 0; linear: zero coordinates).
//  mm: midrange codes (sk_common.cuh) subtracted from the points in modes 0
//  and 2, or null; mm_stride: 0 (one centre) or 2d (per sequence).
__global__ void pack_y_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                              int64_t Lp, int D, double coord_scale, int mode,
                              const unsigned long long *__restrict__ mm, int64_t mm_stride,
                              float *__restrict__ out);
__global__ void pack_x_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                              int64_t Lp2, int D, double coord_scale, int mode,
                              const unsigned long long *__restrict__ mm, int64_t mm_stride,
                              float *__restrict__ out);
__global__ void minmax_seq_kernel(const double *__restrict__ X, int64_t n, int64_t L, int d,
                                  unsigned long long *__restrict__ mm);

int launch_d4(const Params &, int M, int order, int variant, size_t smem, cudaStream_t st);
int launch_d8(const Params &, int M, int order, int variant, size_t smem, cudaStream_t st);
int launch_d16(const Params &, int M, int order, int variant, size_t smem, cudaStream_t st);

// Compiled (n_levels, order) combinations: order 1 with n_levels 1..8, and
// every order 2 <= p <= n_levels for n_levels 2..5 (p = n_levels: geometric).
__host__ __device__ constexpr bool fast_orders_supported(int M, int order) {
  return (order == 1 && M >= 1 && M <= 8) || (order >= 2 && order <= M && M <= 5) ||
         (order == 2 && M <= 8) || (order == 3 && M == 6);
}
__host__ __device__ constexpr int columns_per_lane(int order) { return order == 1 ? 8 : 4; }

template <class LS>
int launch_kernel(const Params &P, size_t smem, cudaStream_t st) {
  using K = void (*)(const Params);
  const K k = P.npanel > 1 ? gram_kernel<LS, true> : gram_kernel<LS, false>;
  SK_CHECK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SK_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NTHREADS, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (P.npanel > 1) cap = std::min<int64_t>(cap, P.max_ctas);  // carry buffer is sized per CTA
  const int grid = (int)std::min<int64_t>(P.ntiles, cap);
  if (grid <= 0) return SK_OK;
  k<<<grid, NTHREADS, smem, st>>>(P);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

// variant: 0 rbf, 1 linear, 2 stationary kinds (StatPointStage, order 1 only),
// 3 rbf with difference=False
template <int D, int LIN>
int launch_impl_lin(const Params &P, int M, int order, size_t smem, cudaStream_t st) {
  if (order == 1) {
    switch (M) {
      case 1: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 1>>(P, smem, st);
      case 2: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 2>>(P, smem, st);
      case 3: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 3>>(P, smem, st);
      case 4: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 4>>(P, smem, st);
      case 5: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 5>>(P, smem, st);
      case 6: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 6>>(P, smem, st);
      case 7: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 7>>(P, smem, st);
      case 8: return launch_kernel<LaneState1<PointStage<D, 8, LIN>, 8>>(P, smem, st);
      default: break;
    }
  } else {
#define SK_G(MM, PP) \
  if (M == MM && order == PP) return launch_kernel<LaneStateG<PointStage<D, 4, LIN>, MM, PP>>(P, smem, st);
    SK_G(2, 2) SK_G(3, 2) SK_G(3, 3) SK_G(4, 2) SK_G(4, 3) SK_G(4, 4)
    SK_G(5, 2) SK_G(5, 3) SK_G(5, 4) SK_G(5, 5) SK_G(6, 2) SK_G(6, 3) SK_G(7, 2) SK_G(8, 2)
#undef SK_G
  }
  return fail(SK_ERR_UNSUPPORTED, "fast path: (n_levels, order) not compiled");
}

template <int D>
int launch_impl_stat(const Params &P, int M, int order, size_t smem, cudaStream_t st) {
  if (order == 1) {
    switch (M) {
      case 1: return launch_kernel<LaneState1<StatPointStage<D, 8>, 1>>(P, smem, st);
      case 2: return launch_kernel<LaneState1<StatPointStage<D, 8>, 2>>(P, smem, st);
      case 3: return launch_kernel<LaneState1<StatPointStage<D, 8>, 3>>(P, smem, st);
      case 4: return launch_kernel<LaneState1<StatPointStage<D, 8>, 4>>(P, smem, st);
      case 5: return launch_kernel<LaneState1<StatPointStage<D, 8>, 5>>(P, smem, st);
      case 6: return launch_kernel<LaneState1<StatPointStage<D, 8>, 6>>(P, smem, st);
      case 7: return launch_kernel<LaneState1<StatPointStage<D, 8>, 7>>(P, smem, st);
      case 8: return launch_kernel<LaneState1<StatPointStage<D, 8>, 8>>(P, smem, st);
      default: break;
    }
  } else {
#define SK_GS(MM, PP) \
  if (M == MM && order == PP) return launch_kernel<LaneStateG<StatPointStage<D, 4>, MM, PP>>(P, smem, st);
    SK_GS(2, 2) SK_GS(3, 2) SK_GS(3, 3) SK_GS(4, 2) SK_GS(4, 3) SK_GS(4, 4)
    SK_GS(5, 2) SK_GS(5, 3) SK_GS(5, 4) SK_GS(5, 5) SK_GS(6, 2) SK_GS(6, 3) SK_GS(7, 2) SK_GS(8, 2)
#undef SK_GS
  }
  return fail(SK_ERR_UNSUPPORTED, "fast path: (n_levels, order) not compiled");
}

// Instantiation helper shared by the per-D translation units.
template <int D>
int launch_impl(const Params &P, int M, int order, int variant, size_t smem, cudaStream_t st) {
  if (variant == 2) return launch_impl_stat<D>(P, M, order, smem, st);
  if (variant == 3) return launch_impl_lin<D, 2>(P, M, order, smem, st);
  return variant == 1 ? launch_impl_lin<D, 1>(P, M, order, smem, st)
                      : launch_impl_lin<D, 0>(P, M, order, smem, st);
}

}  // namespace fast
}  // namespace sk
