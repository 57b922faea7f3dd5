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
// m = 1..M-1. Rows are streamed top to bottom, but lane q runs q steps
// behind lane 0 (a wavefront). That skew turns the 2-D exclusive prefix
//   S_m(i, j) = sum_{i' < i, j' < j} R_m(i', j')
// into a chain: lane q receives from lane q-1 (one __shfl_up per level per
// step) the prefix of everything left of its columns for the SAME row, adds
// its own colaccs serially, and passes the result on next step. Per cell and
// level that is one FADD (scan) + one FFMA (colacc += A * S), i.e. the
// north-star flop model's 4 flops/level/cell, with the cross-lane scan cost
// amortised over C cells.
//
// Pairs stream back to back: a segment keeps its y sequence and walks a
// range of x sequences; each lane switches to the next x when its own row
// counter wraps, so there is no wavefront fill/drain per pair. The level
// sums of a finished pair arrive for free at the segment's last lane: at a
// lane's first step of the next pair, the chain carries sum over all lanes of
// sum_g colacc_m(g) = k_m (and k_M rides a separate chain).
//
// Increments: lane q needs D(g) = G(i,g) - G(i-1,g) for g = C*q - 1, which
// lane q-1 computed one step earlier; it arrives with the carries, so every
// point-kernel value is computed exactly once. Columns beyond L_y repeat the
// last y point (zero increments, A = 0), which is exact.
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

namespace sk {
namespace fast {

constexpr int NWARPS = 8;
constexpr int NTHREADS = NWARPS * 32;
constexpr int C = 8;  // point-kernel columns per lane
constexpr int NSLOT = 3;

struct Params {
  const float *xs;  // x role (Gram rows), packed [nx][lxp][DP]
  const float *ys;  // y role (Gram columns), packed [ny][lyp][DP]
  int64_t nx, ny;
  int lx;        // x points per sequence (rows streamed per pair)
  int lxp, lyp;  // packed point strides
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
  float *carry;  // [max_ctas * NWARPS][rx + 2 jobs][lx rows][nhp]
  int nhp;       // floats per carry entry (NCA chain values, lastD, kout; padded to 4)
  int max_ctas;  // grid size the carry buffer was sized for
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__device__ __forceinline__ void stage_sequence(float *dst, const float *src, int nfloats) {
  for (int k = threadIdx.x * 4; k < nfloats; k += NTHREADS * 4) cp_async16(dst + k, src + k);
  cp_async_commit();
}

template <int M>
__device__ __forceinline__ void write_pair(const Params &P, int64_t i, int64_t j,
                                           const float (&cout)[(M >= 2) ? M - 1 : 1],
                                           float kout) {
  double lv[M + 1];
  lv[0] = 1.0;
#pragma unroll
  for (int m = 1; m < M; ++m) lv[m] = (double)cout[m - 1];
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
  if (P.levels) {
#pragma unroll
    for (int m = 0; m <= M; ++m) P.levels[(row * P.ldk + j) * (M + 1) + m] = lv[m];
    if (mirror) {
#pragma unroll
      for (int m = 0; m <= M; ++m) P.levels[(j * P.ldk + i) * (M + 1) + m] = lv[m];
    }
  }
  if (P.K) {
    const double v = finish_entry(lv, M, P.norm, P.diag_x ? P.diag_x + i * (M + 1) : nullptr,
                                  P.diag_y ? P.diag_y + j * (M + 1) : nullptr);
    P.K[row * P.ldk + j] = v;
    if (mirror) P.K[j * P.ldk + i] = v;
  }
}

// Per-lane register state of one segment lane and the systolic step.
template <int D, int M, bool LINEAR>
struct LaneState {
  static constexpr int DP = D + 4;
  static constexpr int NCA = (M >= 2) ? M - 1 : 0;  // column-accumulated levels 1..M-1
  static constexpr int NCR = (NCA > 0) ? NCA : 1;

  float yv[C][D];
  float yn[C];
  float colacc[NCR][C];
  float prevG[C];
  float cout[NCR];
  float kM, kout, lastD;

  __device__ __forceinline__ void reset_pair() {
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int m = 0; m < NCR; ++m) colacc[m][c] = 0.f;
    }
    kM = 0.f;
  }

  // One row of this lane's C columns. KCHAIN: also run the level-M chain
  // (only needed while some lane of the segment is at a pair boundary).
  //  MULTI: the chain head takes its inputs from `hin` (the previous panel's
  //         carries for this row) when head_buf, instead of zeros
  template <bool KCHAIN, bool MULTI>
  __device__ __forceinline__ void step(const float *__restrict__ xptr, int sw, bool first_lane,
                                       const float *hin, bool head_buf) {
    constexpr unsigned FULL = 0xffffffffu;
    const bool from_buf = MULTI && head_buf;
    // (a) chain values produced by lane q-1 on the previous step
    float dl_raw = __shfl_up_sync(FULL, lastD, 1, sw);
    float cin[NCR];
#pragma unroll
    for (int m = 0; m < NCA; ++m) {
      const float v = __shfl_up_sync(FULL, cout[m], 1, sw);
      cin[m] = first_lane ? (from_buf ? hin[m] : 0.f) : v;
    }
    if (from_buf && first_lane) dl_raw = hin[NCA];
    if (KCHAIN) {
      const float kin = __shfl_up_sync(FULL, kout, 1, sw);
      kout = (first_lane ? (from_buf ? hin[NCA + 1] : 0.f) : kin) + kM;  // complete at a boundary
    }

    // (b) point-kernel row for this lane's columns
    float g[C];
    {
      float acc[C];
#pragma unroll
      for (int c = 0; c < C; ++c) acc[c] = yn[c];
      const float4 *xr = reinterpret_cast<const float4 *>(xptr);
#pragma unroll
      for (int k4 = 0; k4 < D / 4; ++k4) {
        const float4 xv = xr[k4];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          acc[c] = fmaf(xv.x, yv[c][4 * k4 + 0], acc[c]);
          acc[c] = fmaf(xv.y, yv[c][4 * k4 + 1], acc[c]);
          acc[c] = fmaf(xv.z, yv[c][4 * k4 + 2], acc[c]);
          acc[c] = fmaf(xv.w, yv[c][4 * k4 + 3], acc[c]);
        }
      }
      if (LINEAR) {
#pragma unroll
        for (int c = 0; c < C; ++c) g[c] = acc[c];
      } else {
        const float xn = xptr[D];
#pragma unroll
        for (int c = 0; c < C; ++c) g[c] = ex2_approx(fminf(acc[c] + xn, 0.f));
      }
    }

    // (c) increments of the previous DP row: A = D(g) - D(g-1), D = G(r,.) - G(r-1,.)
    float a[C];
    {
      float dv[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        dv[c] = g[c] - prevG[c];
        prevG[c] = g[c];
      }
      // column -1 of the first panel does not exist (A = 0); a later panel's
      // head gets D of the previous panel's last column through the carry
      const float dl = (first_lane && !from_buf) ? dv[0] : dl_raw;
      a[0] = dv[0] - dl;
#pragma unroll
      for (int c = 1; c < C; ++c) a[c] = dv[c] - dv[c - 1];
      lastD = dv[C - 1];
    }

    // (d) level recursion along the row (p = 1): R_m = A * S(R_{m-1})
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
};

template <int D, int M, bool LINEAR, bool MULTI>
__global__ void __launch_bounds__(NTHREADS, 1) gram_p1_kernel(const Params P) {
  static_assert(D % 4 == 0, "D must be a multiple of 4");
  static_assert(M >= 1, "M >= 1");
  using LS = LaneState<D, M, LINEAR>;
  constexpr int DP = LS::DP;
  extern __shared__ __align__(16) float smem[];
  const int lx = P.lx;
  const int slot_floats = lx * DP;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sw = P.sw;
  const int q = lane & (sw - 1);
  const int seg = warp * (32 / sw) + lane / sw;
  const bool last_lane = (q == sw - 1);
  const bool first_lane = (q == 0);

  LS st;
  for (int64_t tile = blockIdx.x; tile < P.ntiles; tile += gridDim.x) {
    const int64_t ty = tile % P.tiles_y;
    const int64_t tx = tile / P.tiles_y;
    const int64_t ybase = ty * P.segs;
    int64_t x0, njobs;
    if (P.diag_mode) {
      x0 = ybase;
      njobs = min((int64_t)P.segs, P.ny - x0);
    } else {
      x0 = P.row_begin + tx * P.rx;
      njobs = min((int64_t)P.rx, P.row_end - x0);
      if (P.symmetric && x0 > ybase + P.segs - 1) continue;  // CTA-uniform
    }
    const int64_t j = ybase + seg;
    const bool jvalid = j < P.ny;
    const int64_t jj = jvalid ? j : P.ny - 1;

    // carry region of this warp (multi-panel only)
    float *cbuf = MULTI ? P.carry + ((size_t)(blockIdx.x * NWARPS + warp) * (P.rx + 2)) * lx * P.nhp
                        : nullptr;
    const int npanel = MULTI ? P.npanel : 1;
    for (int pnl = 0; pnl < npanel; ++pnl) {
      // this lane's y columns of panel pnl (pre-scaled points and their n-terms)
      {
        const float *yp = P.ys + ((size_t)jj * P.lyp + (size_t)pnl * 32 * C + (size_t)q * C) * DP;
#pragma unroll
        for (int c = 0; c < C; ++c) {
#pragma unroll
          for (int k4 = 0; k4 < D / 4; ++k4) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(yp + c * DP) + k4);
            st.yv[c][4 * k4 + 0] = v.x;
            st.yv[c][4 * k4 + 1] = v.y;
            st.yv[c][4 * k4 + 2] = v.z;
            st.yv[c][4 * k4 + 3] = v.w;
          }
          st.yn[c] = LINEAR ? 0.f : __ldg(yp + c * DP + D);
          st.prevG[c] = 0.f;
        }
      }
      st.reset_pair();
      st.kout = st.lastD = 0.f;
#pragma unroll
      for (int m = 0; m < LS::NCR; ++m) st.cout[m] = 0.f;
      const bool head_buf = MULTI && pnl > 0;          // chain inputs from the previous panel
      const bool tail_buf = MULTI && pnl < npanel - 1;  // chain outputs for the next panel
      const bool last_panel = pnl == npanel - 1;

      __syncthreads();  // previous readers are done with the ring (and the carries are visible)
      stage_sequence(smem, P.xs + (size_t)x0 * P.lxp * DP, slot_floats);

      // head inputs, prefetched one step ahead (lane 0 reads job e, row s)
      constexpr int NHM = LS::NCA + 2;
      float hcur[NHM], hnext[NHM];
#pragma unroll
      for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k] = 0.f;
      auto load_head = [&](float (&h)[NHM], int64_t job, int row) {
        if (head_buf && first_lane) {
          const float *src = cbuf + ((size_t)job * lx + row) * P.nhp;
#pragma unroll
          for (int k = 0; k < NHM; ++k) h[k] = src[k];
        }
      };
      auto store_tail = [&](int64_t job, int row) {
        if (tail_buf && last_lane && job >= 0) {
          float *dst = cbuf + ((size_t)job * lx + row) * P.nhp;
#pragma unroll
          for (int m = 0; m < LS::NCA; ++m) dst[m] = st.cout[m];
          dst[LS::NCA] = st.lastD;
          dst[LS::NCA + 1] = st.kout;
        }
      };
      load_head(hcur, 0, 0);

      // Epoch e streams x_{x0+e}: lane q starts that pair at step s = q (its
      // row 0) and spends steps s < q finishing pair e-1. So pair boundaries
      // only occur in steps s < sw ("phase A"); steps s >= sw are branch-free.
      for (int64_t e = 0; e <= njobs; ++e) {
        cp_async_wait_all();
        __syncthreads();
        if (e + 1 < njobs)
          stage_sequence(smem + ((e + 1) % NSLOT) * slot_floats,
                         P.xs + (size_t)(x0 + e + 1) * P.lxp * DP, slot_floats);
        const float *cur = smem + (e % NSLOT) * slot_floats;
        // before its first pair a lane idles on rows of x_{x0} (slot 0)
        const float *prev = (e == 0) ? smem : smem + ((e + NSLOT - 1) % NSLOT) * slot_floats;
        const int steps = (e < njobs) ? lx : sw;
        const int nA = min(sw, steps);
        for (int s = 0; s < nA; ++s) {
          if (MULTI) load_head(hnext, s + 1 < steps ? e : e + 1, s + 1 < steps ? s + 1 : 0);
          const float *xp = (s < q) ? prev + (lx - q + s) * DP : cur + (s - q) * DP;
          st.template step<true, MULTI>(xp, sw, first_lane, hcur, head_buf);
          if (MULTI) {
            // the segment's last lane is at (job, row) = (e, s - q) or (e - 1, lx - q + s)
            if (s >= q)
              store_tail(e, s - q);
            else
              store_tail(e - 1, lx - q + s);
          }
          if (s == q) {  // this lane's pair boundary: pair e-1 is complete
            if (last_panel && last_lane && e >= 1 && jvalid)
              write_pair<M>(P, x0 + e - 1, j, st.cout, st.kout);
            st.reset_pair();
          }
          if (MULTI) {
#pragma unroll
            for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k];
          }
        }
        const float *xp = cur + (nA - q) * DP;
#pragma unroll 2
        for (int s = nA; s < steps; ++s) {
          if (MULTI) load_head(hnext, s + 1 < steps ? e : e + 1, s + 1 < steps ? s + 1 : 0);
          st.template step<false, MULTI>(xp, sw, first_lane, hcur, head_buf);
          if (MULTI) {
            store_tail(e, s - q);
#pragma unroll
            for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k];
          }
          xp += DP;
        }
      }
    }
  }
}

// Pack (N, L, d) float64 -> [N][Lp][DP] float32 with pre-scaled coordinates,
// zero-padded channels, the n-term in column D, and points beyond L
// repeating the last point.
__global__ void pack_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t d,
                            int64_t Lp, int D, int DP, double coord_scale, int with_norm,
                            float *__restrict__ out);

int launch_d4(const Params &, int M, int linear, size_t smem, cudaStream_t st);
int launch_d8(const Params &, int M, int linear, size_t smem, cudaStream_t st);
int launch_d16(const Params &, int M, int linear, size_t smem, cudaStream_t st);

// Instantiation helper shared by the per-D translation units.
template <int D>
int launch_impl(const Params &P, int M, int linear, size_t smem, cudaStream_t st) {
  using K = void (*)(const Params);
  K k = nullptr;
#define SK_CASE(MM)                                                                       \
  case MM:                                                                                \
    if (P.npanel > 1)                                                                     \
      k = linear ? gram_p1_kernel<D, MM, true, true> : gram_p1_kernel<D, MM, false, true>;  \
    else                                                                                  \
      k = linear ? gram_p1_kernel<D, MM, true, false> : gram_p1_kernel<D, MM, false, false>; \
    break;
  switch (M) {
    SK_CASE(1)
    SK_CASE(2)
    SK_CASE(3)
    SK_CASE(4)
    SK_CASE(5)
    SK_CASE(6)
    SK_CASE(7)
    SK_CASE(8)
    default:
      return fail(SK_ERR_UNSUPPORTED, "fast path: n_levels outside 1..8");
  }
#undef SK_CASE
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

}  // namespace fast
}  // namespace sk
