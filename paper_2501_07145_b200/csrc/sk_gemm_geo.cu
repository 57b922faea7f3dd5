// General-order (1 < p <= M) instances of the GEMM-fed path's DP kernel: the
// fused kernel's (n_levels, order) set (sk_fast.cuh fast_orders_supported),
// rbf and linear. A translation unit of its own so it compiles beside
// sk_gemm.cu.
#include "sk_gemm.cuh"

namespace sk {
namespace gemm {

template <bool LIN>
static int launch_geo(const Params &P, int M, int order, cudaStream_t st) {
  using fast::LaneStateG;
  using S4 = fast::GemmStage<4, LIN>;
#define SK_GG(MM, PP) \
  if (M == MM && order == PP) return launch_dp<LaneStateG<S4, MM, PP>>(P, st);
  SK_GG(2, 2) SK_GG(3, 2) SK_GG(3, 3) SK_GG(4, 2) SK_GG(4, 3) SK_GG(4, 4)
  SK_GG(5, 2) SK_GG(5, 3) SK_GG(5, 4) SK_GG(5, 5) SK_GG(6, 2) SK_GG(6, 3) SK_GG(7, 2) SK_GG(8, 2)
#undef SK_GG
  return fail(SK_ERR_UNSUPPORTED, "gemm path: (n_levels, order) not compiled");
}

int launch_dp_geo(const Params &P, int M, int order, bool lin, cudaStream_t st) {
  return lin ? launch_geo<true>(P, M, order, st) : launch_geo<false>(P, M, order, st);
}

}  // namespace gemm
}  // namespace sk
