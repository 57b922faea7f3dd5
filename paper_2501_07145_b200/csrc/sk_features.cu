// Static feature maps of a fitted rfsf_full state (transform_static_features,
// static/features.py:102-124), float64, for rfsf_exact_gram's lifted level
// Grams (features.py:397-443):
//   rff      phi(x) = (1/sqrt(D)) (cos(W^T x), sin(W^T x))      out_dim 2D
//   rff1d    phi(x) = sqrt(2/D) cos(W^T x + b)                  out_dim D
//   nystroem phi(x) = k(x, Z) @ whiten                           out_dim <= D
// One thread per (point, output column); the nystroem landmark Gram k(x, Z)
// goes through the workspace. Features are written into a strided destination
// so every slot lands at its channel offset of one concatenated buffer.
#include <algorithm>
#include <cmath>

#include "sk_common.cuh"

namespace sk {
namespace {

constexpr int FEAT_THREADS = 256;

__global__ void rff_kernel(const double *__restrict__ X, int64_t npts, int64_t d,
                           const double *__restrict__ W, const double *__restrict__ b,
                           int64_t D, int kind, double *__restrict__ out, int64_t ld_out) {
  const int64_t total = npts * D;
  const double s = kind == SK_FEAT_RFF ? 1.0 / sqrt((double)D) : sqrt(2.0 / (double)D);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / D, k = e % D;
    const double *x = X + p * d;
    double acc = 0.0;
    for (int64_t c = 0; c < d; ++c) acc = fma(x[c], W[c * D + k], acc);
    double *o = out + p * ld_out;
    if (kind == SK_FEAT_RFF) {
      double sn, cs;
      sincos(acc, &sn, &cs);
      o[k] = s * cs;
      o[D + k] = s * sn;
    } else {
      o[k] = s * cos(acc + b[k]);
    }
  }
}

__global__ void landmark_gram_kernel(const double *__restrict__ X, int64_t npts, int64_t d,
                                     const double *__restrict__ Z, int64_t D, StaticF64 S,
                                     double *__restrict__ Kz) {
  const int64_t total = npts * D;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / D, l = e % D;
    Kz[e] = static_eval_f64(S, X + p * d, Z + l * d, (int)d);
  }
}

__global__ void whiten_kernel(const double *__restrict__ Kz, int64_t npts, int64_t D,
                              const double *__restrict__ Wh, int64_t out_dim,
                              double *__restrict__ out, int64_t ld_out) {
  const int64_t total = npts * out_dim;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / out_dim, o = e % out_dim;
    const double *kz = Kz + p * D;
    double acc = 0.0;
    for (int64_t l = 0; l < D; ++l) acc = fma(kz[l], Wh[l * out_dim + o], acc);
    out[p * ld_out + o] = acc;
  }
}

unsigned grid_for(int64_t total) {
  return (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((total + FEAT_THREADS - 1) / FEAT_THREADS, (int64_t)sm_count() * 16));
}

}  // namespace

size_t static_features_workspace_bytes(const sk_feature_map &f, int64_t npts) {
  if (f.kind != SK_FEAT_NYSTROEM) return 0;
  return (size_t)std::max<int64_t>(npts, 0) * f.n_components * sizeof(double);
}

int static_features(const sk_feature_map &f, const double *X, int64_t npts, int64_t d,
                    double *out, int64_t ld_out, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (npts <= 0) return SK_OK;
  const int64_t D = f.n_components;
  if (f.kind == SK_FEAT_RFF || f.kind == SK_FEAT_RFF1D) {
    rff_kernel<<<grid_for(npts * D), FEAT_THREADS, 0, st>>>(X, npts, d, f.weights, f.phases, D,
                                                           f.kind, out, ld_out);
    SK_CHECK_LAUNCH();
    return SK_OK;
  }
  const size_t need = static_features_workspace_bytes(f, npts);
  if (!ws || ws_bytes < need)
    return fail(SK_ERR_WORKSPACE, "workspace too small for the nystroem map: need " +
                                      std::to_string(need) + " bytes");
  double *Kz = (double *)ws;
  landmark_gram_kernel<<<grid_for(npts * D), FEAT_THREADS, 0, st>>>(X, npts, d, f.landmarks, D,
                                                                   to_static(f.base), Kz);
  SK_CHECK_LAUNCH();
  whiten_kernel<<<grid_for(npts * f.out_dim), FEAT_THREADS, 0, st>>>(Kz, npts, D, f.whiten,
                                                                    f.out_dim, out, ld_out);
  SK_CHECK_LAUNCH();
  return SK_OK;
}

}  // namespace sk
