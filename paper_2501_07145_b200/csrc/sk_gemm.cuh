// The GEMM-fed path's DP kernel template (sk_gemm.cu): shared by the
// order-1 instances (sk_gemm.cu) and the general-order ones (sk_gemm_geo.cu,
// a separate translation unit so the two compile in parallel).
#pragma once
#include <algorithm>

#include "sk_fast.cuh"

namespace sk {
namespace gemm {

using fast::NTHREADS;
using fast::NWARPS;
using fast::Params;

// The fused kernel's epoch/panel structure without the shared-memory x ring:
// every lane addresses its pair's rows in the cell matrix directly.
template <class LS, bool MULTI>
__global__ void __launch_bounds__(NTHREADS) gemm_dp_kernel(const Params P) {
  constexpr int M = LS::M;
  constexpr int C = LS::C;
  const int lx2 = P.lx2;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sw = P.sw;
  const int q = lane & (sw - 1);
  const int seg = warp * (32 / sw) + lane / sw;
  const bool last_lane = (q == sw - 1);
  const bool first_lane = (q == 0);
  const int64_t rowpair = 2 * P.s_ld;  // floats between row pairs

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
      if (P.symmetric && x0 > ybase + P.segs - 1) continue;
    }
    const int64_t j = ybase + seg;
    const bool jvalid = j < P.ny;
    const int64_t jj = jvalid ? j : P.ny - 1;
    // row 0 of pair (x, jj) at this lane's first column of panel 0
    auto pair_base = [&](int64_t x) -> const float * {
      const int64_t xl = min(max(x, x0), x0 + njobs - 1) - P.x_blk0;
      return P.S + xl * P.s_xstride + jj * P.s_ystride + (int64_t)q * C;
    };
    float *cbuf = MULTI ? P.carry + ((size_t)(blockIdx.x * NWARPS + warp) * (P.rx + 2)) * lx2 * P.nhp
                        : nullptr;
    const int npanel = MULTI ? P.npanel : 1;
    for (int pnl = 0; pnl < npanel; ++pnl) {
      const int64_t pcol = (int64_t)pnl * 32 * C;
      st.reset_y();
      st.reset_panel();
      const bool head_buf = MULTI && pnl > 0;
      const bool tail_buf = MULTI && pnl < npanel - 1;
      const bool last_panel = pnl == npanel - 1;
      if (MULTI) __syncwarp();  // carries of the previous panel (same warp) are visible
      constexpr int NHM = LS::NHP;
      float hcur[NHM], hnext[NHM];
#pragma unroll
      for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k] = 0.f;
      auto load_head = [&](float (&h)[NHM], int64_t job, int rp) {
        if (head_buf) fast::load_f4(h, cbuf + ((size_t)job * lx2 + rp) * P.nhp);
      };
      auto store_tail = [&](int64_t job, int rp) {
        st.store_carry(cbuf + ((size_t)job * lx2 + rp) * P.nhp, tail_buf && last_lane && job >= 0);
      };
      load_head(hcur, 0, 0);
      for (int64_t e = 0; e <= njobs; ++e) {
        const float *cur = pair_base(x0 + e) + pcol;
        const float *prev = pair_base(e == 0 ? x0 : x0 + e - 1) + pcol;
        const int steps = (e < njobs) ? lx2 : sw;
        const int nA = min(sw, steps);
        for (int s = 0; s < nA; ++s) {
          if (MULTI) load_head(hnext, s + 1 < steps ? e : e + 1, s + 1 < steps ? s + 1 : 0);
          const float *xp = (s < q) ? prev + (int64_t)(lx2 - q + s) * rowpair
                                    : cur + (int64_t)(s - q) * rowpair;
          st.template step<true, MULTI, true>(xp, sw, first_lane, hcur, head_buf, s == q);
          if (MULTI) {
            if (s >= q)
              store_tail(e, s - q);
            else
              store_tail(e - 1, lx2 - q + s);
          }
          if (s == q && last_panel && last_lane && e >= 1 && jvalid)
            fast::write_pair<M>(P, x0 + e - 1, j, st.level_sums(), st.kout);
          if (MULTI) {
#pragma unroll
            for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k];
          }
        }
        const float *xp = cur + (int64_t)(nA - q) * rowpair;
#pragma unroll 2
        for (int s = nA; s < steps; ++s) {
          if (MULTI) load_head(hnext, s + 1 < steps ? e : e + 1, s + 1 < steps ? s + 1 : 0);
          st.template step<false, MULTI, false>(xp, sw, first_lane, hcur, head_buf, false);
          if (MULTI) {
            store_tail(e, s - q);
#pragma unroll
            for (int k = 0; k < NHM; ++k) hcur[k] = hnext[k];
          }
          xp += rowpair;
        }
      }
    }
  }
}

template <class LS, bool SINGLE = false>
inline int launch_dp(const Params &P, cudaStream_t st) {
  using K = void (*)(const Params);
  K k;
  if constexpr (SINGLE)
    k = gemm_dp_kernel<LS, false>;
  else
    k = P.npanel > 1 ? gemm_dp_kernel<LS, true> : gemm_dp_kernel<LS, false>;
  int per_sm = 0;
  SK_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NTHREADS, 0));
  if (per_sm < 1) per_sm = 1;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (P.npanel > 1) cap = std::min<int64_t>(cap, P.max_ctas);
  const int grid = (int)std::min<int64_t>(P.ntiles, cap);
  if (grid <= 0) return SK_OK;
  k<<<grid, NTHREADS, 0, st>>>(P);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

// general order 1 < p <= M (sk_gemm_geo.cu)
int launch_dp_geo(const Params &P, int M, int order, bool lin, cudaStream_t st);

}  // namespace gemm
}  // namespace sk
