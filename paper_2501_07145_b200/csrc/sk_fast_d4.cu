// Fused FP32 kernels instantiated for 4 padded channels (n_levels 1..8, rbf/linear).
#include "sk_fast.cuh"

namespace sk {
namespace fast {
int launch_d4(const Params &P, int M, int order, int variant, size_t smem, cudaStream_t st) {
  return launch_impl<4>(P, M, order, variant, smem, st);
}
}  // namespace fast
}  // namespace sk
