// C ABI of libsigkern_b200 (include/sigkern_b200.h): validation and dispatch
// between the fused FP32 kernels and the general float64 kernel.
#include <algorithm>
#include <string>

#include "sk_common.cuh"

namespace sk {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string &msg) { g_error = msg; }
void clear_error() { g_error.clear(); }

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

namespace {

int check_config(const sk_kernel_config *c) {
  if (!c) return fail(SK_ERR_INVALID, "config is NULL");
  const sk_static_spec &s = c->static_spec;
  if (s.kind < SK_LINEAR || s.kind > SK_RATIONAL_QUADRATIC)
    return fail(SK_ERR_INVALID, "unknown kernel kind " + std::to_string(s.kind));
  if (!(s.scale > 0)) return fail(SK_ERR_INVALID, "scale must be positive");
  if (s.degree < 1) return fail(SK_ERR_INVALID, "degree must be a positive integer");
  if (!(s.bandwidth > 0)) return fail(SK_ERR_INVALID, "bandwidth must be positive");
  if (!(s.alpha > 0)) return fail(SK_ERR_INVALID, "alpha must be positive");
  if (c->n_levels < 0) return fail(SK_ERR_INVALID, "n_levels must be a non-negative integer");
  if (c->order < 1 || c->order > std::max(1, c->n_levels))
    return fail(SK_ERR_INVALID, "order must be the effective order in [1, max(1, n_levels)]");
  if (c->normalization < SK_NORM_NONE || c->normalization > SK_NORM_GLOBAL)
    return fail(SK_ERR_INVALID, "normalization must be none/levelwise/global");
  if (c->precision != SK_PREC_FP32 && c->precision != SK_PREC_FP64)
    return fail(SK_ERR_INVALID, "precision must be SK_PREC_FP32 or SK_PREC_FP64");
  if (c->flags & ~SK_FLAG_NO_FIXUP) return fail(SK_ERR_INVALID, "unknown flags");
  return SK_OK;
}

int check_static(const sk_static_spec *sp) {
  if (!sp) return fail(SK_ERR_INVALID, "spec is NULL");
  if (sp->kind < SK_LINEAR || sp->kind > SK_RATIONAL_QUADRATIC)
    return fail(SK_ERR_INVALID, "unknown kernel kind " + std::to_string(sp->kind));
  if (!(sp->scale > 0)) return fail(SK_ERR_INVALID, "scale must be positive");
  if (sp->degree < 1) return fail(SK_ERR_INVALID, "degree must be a positive integer");
  if (!(sp->bandwidth > 0)) return fail(SK_ERR_INVALID, "bandwidth must be positive");
  if (!(sp->alpha > 0)) return fail(SK_ERR_INVALID, "alpha must be positive");
  return SK_OK;
}

int check_pde_len(int64_t l, int difference) {
  if (difference && l < 2) return fail(SK_ERR_INVALID, "pde kernel needs at least one increment per sequence");
  return SK_OK;
}

int check_generic_limits(const sk_kernel_config &c) {
  if (c.n_levels > GEN_MAX_LEVELS)
    return fail(SK_ERR_UNSUPPORTED, "n_levels > " + std::to_string(GEN_MAX_LEVELS) +
                                        " is not compiled into the float64 kernel");
  if (c.order > GEN_MAX_ORDER)
    return fail(SK_ERR_UNSUPPORTED, "order > " + std::to_string(GEN_MAX_ORDER) +
                                        " is not compiled into the float64 kernel");
  return SK_OK;
}

// float64 path: the CTA-per-pair row-scan kernel at order 1 once rows have
// >= 32 increments (below that most of a CTA would idle), else thread per pair
// the row-scan kernels (warp-per-pair for short rows, CTA-per-pair beyond) or,
// for short sequences outside the warp kernel's range, the generic kernel
bool use_rowscan(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config &c) {
  const int64_t T2 = c.difference ? ly - 1 : ly;
  return rowscan_supported(lx, ly, c) && (T2 >= 32 || warp_gram_ok(lx, ly, d, c));
}

constexpr int64_t SELF64_MAX_L = 32;  // float64 general-order self levels up to this length

int effective_order(const sk_kernel_config &c) {
  return std::max(1, std::min(c.order, std::max(c.n_levels, 1)));
}

int self_fixup(const double *X, int64_t n, int64_t l, int64_t d, const sk_kernel_config &c,
               double *out, void *ws, size_t ws_bytes, cudaStream_t st) {
  if (rowscan_supported(l, l, c)) return cert_self_fixup(X, n, l, d, c, out, ws, ws_bytes, st);
  return fp64_self_fixup(X, n, l, d, c, out, ws, ws_bytes, st);
}

int check_batch(const double *X, int64_t n, int64_t l, int64_t d, const char *what) {
  if (n < 0 || l < 1 || d < 1)
    return fail(SK_ERR_INVALID, std::string(what) + ": expected an (N, L, d) batch with L, d >= 1");
  if (n > 0 && !X) return fail(SK_ERR_INVALID, std::string(what) + " is NULL");
  return SK_OK;
}

}  // namespace
}  // namespace sk

using namespace sk;

extern "C" {

int sk_abi_version(void) { return SK_ABI_VERSION; }

const char *sk_last_error(void) { return g_error.c_str(); }

int sk_fast_path(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config *cfg) {
  if (!cfg) return 0;
  return path_of(lx, ly, d, *cfg);
}

size_t sk_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                          const sk_kernel_config *cfg) {
  if (!cfg) return 0;
  // the largest need of the calls a Gram makes: self levels of X and of Y
  // (normalisation) and the Gram itself, each on the path it dispatches to
  auto use = [&](int64_t n1, int64_t l1, int64_t n2, int64_t l2) -> size_t {
    const int path = n2 > 0 ? path_of(l1, l2, d, *cfg) : path_of(l1, l1, d, *cfg);
    // FP32 paths: the float64 fix-up reuses the same workspace afterwards
    // (Gram: after the FP32 level-1 buffer of the certification)
    const int64_t l2e = n2 > 0 ? l2 : l1;
    const int64_t n2e = n2 > 0 ? n2 : n1;
    // float64 self levels at general order (sk_self_levels), unless SK_FLAG_NO_FIXUP
    const size_t self64 = (n2 == 0 && effective_order(*cfg) > 1 && l1 <= SELF64_MAX_L &&
                           (path == 1 || path == 2))
                              ? generic_workspace_bytes(n1, l1, l1, *cfg)
                              : 0;
    const size_t fix = rowscan_supported(l1, l2e, *cfg)
                           ? cert_workspace_bytes(n1, l1, n2e, l2e, d, *cfg)
                           : fixup_workspace_bytes(l1, l2e, *cfg);
    const size_t k1 = n2 > 0 ? k1buf_bytes(n1, n2, cfg->normalization) : 0;
    if (path == 1)
      return std::max(self64, k1 + std::max(fix, fast_workspace_bytes(n1, l1, n2, l2, d, *cfg)));
    if (path == 2)
      return std::max(self64, k1 + std::max(fix, gemm_workspace_bytes(n1, l1, n2, l2, d, *cfg)));
    return n2 > 0 ? std::max(generic_workspace_bytes(n1 * n2, l1, l2, *cfg),
                             rowscan_workspace_bytes(n1 * n2, l1, l2, *cfg))
                  : std::max(generic_workspace_bytes(n1, l1, l1, *cfg),
                             rowscan_workspace_bytes(n1, l1, l1, *cfg));
  };
  size_t need = use(nx, lx, 0, 0);
  if (ny > 0) need = std::max({need, use(ny, ly, 0, 0), use(nx, lx, ny, ly)});
  return need;
}

int sk_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                   const sk_kernel_config *cfg, double *out, void *workspace,
                   size_t workspace_bytes, void *stream) {
  clear_error();
  int rc = check_config(cfg);
  if (rc) return rc;
  if ((rc = check_batch(X, n, l, d, "X"))) return rc;
  if (n > 0 && !out) return fail(SK_ERR_INVALID, "out is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const bool fix = !(cfg->flags & SK_FLAG_NO_FIXUP);
  // General order (p > 1), short sequences: the FP32 self levels' high levels
  // carried up to ~2e-5 relative error at L = 13 (tools/path_sweep.py), which
  // the normalisation passes on to every entry of the row; up to SELF64_MAX_L
  // points the float64 kernel costs little (the thread-per-pair kernel at
  // L = 128 would be 8x the Gram's time), so they are computed in float64.
  if (fix && effective_order(*cfg) > 1 && cfg->precision == SK_PREC_FP32 &&
      l <= SELF64_MAX_L && (fast_supported(l, l, d, *cfg) || gemm_supported(l, l, d, *cfg))) {
    if ((rc = check_generic_limits(*cfg))) return rc;
    return generic_self_levels(X, n, l, d, *cfg, out, workspace, workspace_bytes, st);
  }
  if (fast_supported(l, l, d, *cfg)) {
    rc = fast_self_levels(X, n, l, d, *cfg, out, workspace, workspace_bytes, st);
    if (!rc && fix) rc = self_fixup(X, n, l, d, *cfg, out, workspace, workspace_bytes, st);
    return rc;
  }
  if (gemm_supported(l, l, d, *cfg)) {
    rc = gemm_self_levels(X, n, l, d, *cfg, out, workspace, workspace_bytes, st);
    if (!rc && fix) rc = self_fixup(X, n, l, d, *cfg, out, workspace, workspace_bytes, st);
    return rc;
  }
  if ((rc = check_generic_limits(*cfg))) return rc;
  if (use_rowscan(l, l, d, *cfg))
    return rowscan_gram(X, n, l, X, n, l, d, 2, *cfg, 0, n, nullptr, nullptr, nullptr, 0, nullptr,
                        out, workspace, workspace_bytes, st);
  return generic_self_levels(X, n, l, d, *cfg, out, workspace, workspace_bytes, st);
}

int sk_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
            int64_t d, int32_t symmetric, const sk_kernel_config *cfg, int64_t row_begin,
            int64_t row_end, const double *diag_x, const double *diag_y, double *K,
            int64_t ldk, double *levels, void *workspace, size_t workspace_bytes,
            void *stream) {
  clear_error();
  int rc = check_config(cfg);
  if (rc) return rc;
  if ((rc = check_batch(X, nx, lx, d, "X"))) return rc;
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  } else if ((rc = check_batch(Y, ny, ly, d, "Y"))) {
    return rc;
  }
  if (row_begin < 0 || row_end > nx || row_begin > row_end)
    return fail(SK_ERR_INVALID, "row range outside [0, nx]");
  if (!K && !levels) return fail(SK_ERR_INVALID, "neither K nor levels requested");
  if (ldk < ny) return fail(SK_ERR_INVALID, "ldk < ny");
  if (cfg->normalization != SK_NORM_NONE && (!diag_x || (!symmetric && !diag_y)))
    return fail(SK_ERR_INVALID, "normalization needs diag_x and diag_y self levels");
  cudaStream_t st = (cudaStream_t)stream;
  const int path = path_of(lx, ly, d, *cfg);
  if (path != 0) {
    // FP32 paths: [level-1 buffer of the certification | path workspace]
    const size_t k1b = k1buf_bytes(nx, ny, cfg->normalization);
    if (!workspace || workspace_bytes < k1b)
      return fail(SK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(k1b) + "+");
    float *k1 = K ? (float *)workspace : nullptr;
    void *ws = (char *)workspace + k1b;
    const size_t wsb = workspace_bytes - k1b;
    const double *dy = symmetric ? diag_x : diag_y;
    if (path == 1)
      rc = fast_gram(X, nx, lx, Y, ny, ly, d, symmetric, *cfg, row_begin, row_end, diag_x, dy, K,
                     ldk, levels, k1, ws, wsb, st);
    else
      rc = gemm_gram(X, nx, lx, Y, ny, ly, d, symmetric, *cfg, row_begin, row_end, diag_x, dy, K,
                     ldk, levels, k1, ws, wsb, st);
    // certification pass: uncertified entries -> float64, exact level 1
    if (!rc && K && !(cfg->flags & SK_FLAG_NO_FIXUP)) {
      if (rowscan_supported(lx, ly, *cfg))
        rc = cert_fixup(X, nx, lx, Y, ny, ly, d, symmetric, *cfg, row_begin, row_end, diag_x, dy,
                        k1, K, ldk, levels, ws, wsb, st);
      else
        rc = fp64_fixup(X, nx, lx, Y, ny, ly, d, symmetric, *cfg, row_begin, row_end, diag_x, dy,
                        k1, K, ldk, levels, ws, wsb, st);
    }
    return rc;
  }
  if ((rc = check_generic_limits(*cfg))) return rc;
  if (use_rowscan(lx, ly, d, *cfg))
    return rowscan_gram(X, nx, lx, Y, ny, ly, d, symmetric ? 1 : 0, *cfg, row_begin, row_end,
                        diag_x, symmetric ? diag_x : diag_y, K, ldk, levels, nullptr, workspace,
                        workspace_bytes, st);
  return generic_gram(X, nx, lx, Y, ny, ly, d, symmetric, *cfg, row_begin, row_end, diag_x,
                      symmetric ? diag_x : diag_y, K, ldk, levels, workspace, workspace_bytes,
                      st);
}

size_t sk_levels_dp_workspace_bytes(int64_t batch, int64_t t1, int64_t t2, int32_t n_levels,
                                    int32_t order) {
  (void)t1;
  return generic_levels_dp_workspace_bytes(batch, t2, n_levels, order);
}

int sk_levels_dp(const double *A, int64_t batch, int64_t t1, int64_t t2, int32_t n_levels,
                 int32_t order, int32_t per_level, double *out, void *workspace,
                 size_t workspace_bytes, void *stream) {
  clear_error();
  if (batch < 0 || t1 < 0 || t2 < 0) return fail(SK_ERR_INVALID, "negative shape");
  if (n_levels < 0) return fail(SK_ERR_INVALID, "n_levels must be a non-negative integer");
  if (order < 1) return fail(SK_ERR_INVALID, "order must be a positive integer");
  if (n_levels > GEN_MAX_LEVELS)
    return fail(SK_ERR_UNSUPPORTED, "n_levels > " + std::to_string(GEN_MAX_LEVELS));
  if (std::min(order, std::max(n_levels, 1)) > GEN_MAX_ORDER)
    return fail(SK_ERR_UNSUPPORTED, "order > " + std::to_string(GEN_MAX_ORDER));
  if (batch > 0 && (!out || (!A && t1 * t2 > 0))) return fail(SK_ERR_INVALID, "NULL pointer");
  return generic_levels_from_increments(A, batch, t1, t2, n_levels, order, per_level, out,
                                        workspace, workspace_bytes, (cudaStream_t)stream);
}

int sk_increment_tensor(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                        int64_t ly, int64_t d, int32_t paired, const sk_static_spec *spec,
                        int32_t difference, double *out, void *stream) {
  clear_error();
  if (!spec) return fail(SK_ERR_INVALID, "spec is NULL");
  int rc;
  if ((rc = check_batch(X, nx, lx, d, "X"))) return rc;
  if ((rc = check_batch(Y, ny, ly, d, "Y"))) return rc;
  if (paired && nx != ny) return fail(SK_ERR_INVALID, "paired increments need nx == ny");
  return increment_tensor(X, nx, lx, Y, ny, ly, d, paired, *spec, difference, out,
                          (cudaStream_t)stream);
}

int sk_pairwise_dist(const double *X, int64_t n, int64_t d, double *out, void *stream) {
  clear_error();
  if (n < 0 || d < 1) return fail(SK_ERR_INVALID, "expected (n, d) points with d >= 1");
  if (n > 1 && (!X || !out)) return fail(SK_ERR_INVALID, "NULL pointer");
  return pairwise_dist(X, n, d, out, (cudaStream_t)stream);
}

size_t sk_pde_workspace_bytes(int64_t npairs, int64_t ly, int32_t difference) {
  return pde_workspace_bytes(npairs, ly, difference);
}

int sk_pde_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny, int64_t ly,
                int64_t d, int32_t symmetric, const sk_static_spec *spec, int32_t difference,
                int64_t row_begin, int64_t row_end, double *K, int64_t ldk, void *workspace,
                size_t workspace_bytes, void *stream) {
  clear_error();
  int rc;
  if ((rc = check_static(spec))) return rc;
  if ((rc = check_batch(X, nx, lx, d, "X"))) return rc;
  if (symmetric) {
    Y = X;
    ny = nx;
    ly = lx;
  } else if ((rc = check_batch(Y, ny, ly, d, "Y"))) {
    return rc;
  }
  if ((rc = check_pde_len(lx, difference)) || (rc = check_pde_len(ly, difference))) return rc;
  if (row_begin < 0 || row_end > nx || row_begin > row_end)
    return fail(SK_ERR_INVALID, "row range outside [0, nx]");
  if (!K) return fail(SK_ERR_INVALID, "K is NULL");
  if (ldk < ny) return fail(SK_ERR_INVALID, "ldk < ny");
  return pde_gram(X, nx, lx, Y, ny, ly, d, symmetric, *spec, difference, row_begin, row_end, K,
                  ldk, workspace, workspace_bytes, (cudaStream_t)stream);
}

int sk_pde_self(const double *X, int64_t n, int64_t l, int64_t d, const sk_static_spec *spec,
                int32_t difference, double *out, void *workspace, size_t workspace_bytes,
                void *stream) {
  clear_error();
  int rc;
  if ((rc = check_static(spec))) return rc;
  if ((rc = check_batch(X, n, l, d, "X"))) return rc;
  if ((rc = check_pde_len(l, difference))) return rc;
  if (n > 0 && !out) return fail(SK_ERR_INVALID, "out is NULL");
  return pde_self(X, n, l, d, *spec, difference, out, workspace, workspace_bytes,
                  (cudaStream_t)stream);
}

size_t sk_static_features_workspace_bytes(const sk_feature_map *map, int64_t npts) {
  return map ? static_features_workspace_bytes(*map, npts) : 0;
}

int sk_static_features(const sk_feature_map *map, const double *X, int64_t npts, int64_t d,
                       double *out, int64_t ld_out, void *workspace, size_t workspace_bytes,
                       void *stream) {
  clear_error();
  if (!map) return fail(SK_ERR_INVALID, "feature map is NULL");
  if (map->kind < SK_FEAT_RFF || map->kind > SK_FEAT_NYSTROEM)
    return fail(SK_ERR_INVALID, "unknown feature kind " + std::to_string(map->kind));
  if (map->reserved != 0) return fail(SK_ERR_INVALID, "reserved must be 0");
  if (map->n_components < 1) return fail(SK_ERR_INVALID, "n_components must be a positive integer");
  const int64_t want = map->kind == SK_FEAT_RFF ? 2 * map->n_components
                       : map->kind == SK_FEAT_RFF1D ? map->n_components : -1;
  if (want >= 0 && map->out_dim != want)
    return fail(SK_ERR_INVALID, "out_dim does not match the feature kind");
  if (map->out_dim < 0 || map->out_dim > std::max<int64_t>(map->n_components, want))
    return fail(SK_ERR_INVALID, "out_dim outside [0, n_components]");
  if (npts < 0 || d < 1) return fail(SK_ERR_INVALID, "expected (npts, d) points with d >= 1");
  if (ld_out < map->out_dim) return fail(SK_ERR_INVALID, "ld_out < out_dim");
  if (npts == 0) return SK_OK;
  if (!X || !out) return fail(SK_ERR_INVALID, "NULL pointer");
  if (map->kind == SK_FEAT_NYSTROEM) {
    int rc;
    if ((rc = check_static(&map->base))) return rc;
    if (!map->landmarks || (map->out_dim > 0 && !map->whiten))
      return fail(SK_ERR_INVALID, "nystroem map needs landmarks and whiten");
  } else if (!map->weights || (map->kind == SK_FEAT_RFF1D && !map->phases)) {
    return fail(SK_ERR_INVALID, "rff map needs weights (and phases for rff1d)");
  }
  return static_features(*map, X, npts, d, out, ld_out, workspace, workspace_bytes,
                         (cudaStream_t)stream);
}

size_t sk_lifted_workspace_bytes(int64_t npairs, int64_t ly, int32_t n_levels, int32_t order,
                                 int32_t difference) {
  return lifted_workspace_bytes(npairs, ly, n_levels, order, difference);
}

size_t sk_lifted_gram_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly,
                                      int32_t n_levels, int32_t order, int32_t difference) {
  if (nx <= 0 || ny <= 0 || lx <= 0 || ly <= 0 || n_levels < 0) return 0;
  return lifted_gram_workspace_bytes(nx, lx, ny, ly, n_levels, order, difference);
}

int sk_lifted_gram(const double *UX, int64_t nx, int64_t lx, const double *UY, int64_t ny,
                   int64_t ly, int64_t width, const int64_t *slot_offsets, int32_t n_levels,
                   int32_t order, int32_t difference, int32_t normalization, int32_t symmetric,
                   int64_t row_begin, int64_t row_end, const double *diag_x,
                   const double *diag_y, double *K, int64_t ldk, double *levels,
                   void *workspace, size_t workspace_bytes, void *stream) {
  clear_error();
  int rc;
  if (n_levels < 0) return fail(SK_ERR_INVALID, "n_levels must be a non-negative integer");
  if (order < 1 || order > std::max(1, (int)n_levels))
    return fail(SK_ERR_INVALID, "order must be the effective order in [1, max(1, n_levels)]");
  if (normalization < SK_NORM_NONE || normalization > SK_NORM_GLOBAL)
    return fail(SK_ERR_INVALID, "normalization must be none/levelwise/global");
  if (!slot_offsets) return fail(SK_ERR_INVALID, "slot_offsets is NULL");
  if ((rc = check_batch(UX, nx, lx, width, "UX"))) return rc;
  if (symmetric) {
    UY = UX;
    ny = nx;
    ly = lx;
  } else if ((rc = check_batch(UY, ny, ly, width, "UY"))) {
    return rc;
  }
  if (row_begin < 0 || row_end > nx || row_begin > row_end)
    return fail(SK_ERR_INVALID, "row range outside [0, nx]");
  if (!K && !levels) return fail(SK_ERR_INVALID, "K and levels are both NULL");
  if (ldk < ny) return fail(SK_ERR_INVALID, "ldk < ny");
  if (normalization != SK_NORM_NONE && (!diag_x || !diag_y))
    return fail(SK_ERR_INVALID, "normalization needs diag_x and diag_y");
  return lifted_gram(UX, nx, lx, UY, ny, ly, width, slot_offsets, n_levels, order, difference,
                     normalization, symmetric, row_begin, row_end, diag_x, diag_y, K, ldk,
                     levels, workspace, workspace_bytes, (cudaStream_t)stream);
}

int sk_lifted_self_levels(const double *UX, int64_t n, int64_t l, int64_t width,
                          const int64_t *slot_offsets, int32_t n_levels, int32_t order,
                          int32_t difference, double *out, void *workspace,
                          size_t workspace_bytes, void *stream) {
  clear_error();
  int rc;
  if (n_levels < 0) return fail(SK_ERR_INVALID, "n_levels must be a non-negative integer");
  if (order < 1 || order > std::max(1, (int)n_levels))
    return fail(SK_ERR_INVALID, "order must be the effective order in [1, max(1, n_levels)]");
  if (!slot_offsets) return fail(SK_ERR_INVALID, "slot_offsets is NULL");
  if ((rc = check_batch(UX, n, l, width, "UX"))) return rc;
  if (n > 0 && !out) return fail(SK_ERR_INVALID, "out is NULL");
  return lifted_self_levels(UX, n, l, width, slot_offsets, n_levels, order, difference, out,
                            workspace, workspace_bytes, (cudaStream_t)stream);
}

}  // extern "C"
