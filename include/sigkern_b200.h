/*
 * sigkern_b200 — C ABI of the B200-native truncated signature-kernel Gram path.
 *
 * This is the drop-in boundary for the reference's dual dynamic-programming
 * path, `sigkern.kernels.sig_kernel_gram(..., algorithm="dp")`
 * (/root/reference/pkg/src/sigkern/kernels.py:530-600), and the two public
 * building blocks it is made of, `increment_tensor` (kernels.py:263-281) and
 * `sig_levels_dp` (kernels.py:144-201).
 *
 * Conventions
 *  - Every array pointer is DEVICE memory owned by the caller; every call is
 *    stream-ordered on `stream` (a cudaStream_t, NULL = legacy default stream).
 *  - Sequence batches are row-major float64 (N, L, d), exactly the reference's
 *    `(N, L, d)` ndarray layout (kernels.py:414-422).
 *  - Kernel values are float64 on output, as in the reference.
 *  - The only scratch is the caller-sized workspace (`sk_workspace_bytes`);
 *    the library never allocates device memory itself.
 *  - Return value: SK_OK or an SK_ERR_* code; `sk_last_error()` holds a
 *    thread-local message. Argument validation mirrors the reference's
 *    ValueError cases; the host wrapper re-raises them with the reference's
 *    exception types and messages.
 *  - Re-entrant per stream; no global mutable state besides the error text.
 */
#ifndef SIGKERN_B200_H
#define SIGKERN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 2

#if defined(__GNUC__)
#define SK_API __attribute__((visibility("default")))
#else
#define SK_API
#endif

enum sk_status {
  SK_OK = 0,
  SK_ERR_INVALID = 1,     /* bad argument (reference: ValueError) */
  SK_ERR_CUDA = 2,        /* CUDA runtime / launch failure */
  SK_ERR_WORKSPACE = 3,   /* workspace too small */
  SK_ERR_UNSUPPORTED = 4  /* configuration outside the compiled kernels */
};

/* Static kernel kinds, in the order of static/kernels.py:25-33. */
enum sk_static_kind {
  SK_LINEAR = 0,
  SK_POLYNOMIAL = 1,
  SK_RBF = 2,
  SK_MATERN12 = 3,
  SK_MATERN32 = 4,
  SK_MATERN52 = 5,
  SK_RATIONAL_QUADRATIC = 6
};

/* KernelConfig.normalization (kernels.py:52). */
enum sk_normalization { SK_NORM_NONE = 0, SK_NORM_LEVELWISE = 1, SK_NORM_GLOBAL = 2 };

/* Arithmetic of the level recursion. FP32: the fused sm_100a kernels
 * (float32 increments and scans, float64 cross-lane level sums); FP64:
 * float64 throughout (bit-level agreement with the reference to ~1e-13). */
enum sk_precision { SK_PREC_FP32 = 0, SK_PREC_FP64 = 1 };

/* StaticKernelSpec (static/kernels.py:39-53). */
typedef struct sk_static_spec {
  int32_t kind;       /* sk_static_kind */
  int32_t degree;     /* polynomial degree */
  double scale;       /* linear/polynomial inner-product scale */
  double gamma;       /* polynomial offset */
  double bandwidth;   /* length scale of the stationary kinds */
  double alpha;       /* rational-quadratic shape */
} sk_static_spec;

/* KernelConfig (kernels.py:59-91). `order` is the EFFECTIVE order
 * (KernelConfig.effective_order, kernels.py:85-91): 1 <= order <= max(1, n_levels). */
typedef struct sk_kernel_config {
  sk_static_spec static_spec;
  int32_t n_levels;
  int32_t order;
  int32_t difference;     /* 1: double-differenced increments, 0: raw point kernel */
  int32_t normalization;  /* sk_normalization */
  int32_t precision;      /* sk_precision */
  int32_t flags;          /* sk_config_flags; 0 = default */
} sk_kernel_config;

/* sk_kernel_config.flags. SK_FLAG_NO_FIXUP (diagnostics): leave the FP32
 * paths' uncertified entries as NaN markers instead of recomputing them in
 * float64 (see sk_gram). */
enum sk_config_flags { SK_FLAG_NO_FIXUP = 1 };

/* Library ABI version (SK_ABI_VERSION). */
SK_API int sk_abi_version(void);

/* Thread-local text of the last error on this host thread ("" if none). */
SK_API const char *sk_last_error(void);

/* Bytes of workspace `sk_gram` / `sk_self_levels` need for these shapes
 * (0 when the float64 path is selected). `ny`/`ly` may be 0 for self levels. */
SK_API size_t sk_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly, int64_t d,
                          const sk_kernel_config *cfg);

/* 1 if `cfg` at these shapes runs on the fused FP32 sm_100a kernels, 0 if it
 * runs on the general float64 kernel. */
SK_API int sk_fast_path(int64_t lx, int64_t ly, int64_t d, const sk_kernel_config *cfg);

/*
 * Self level values k_m(x_i, x_i), m = 0..n_levels, for every sequence:
 * out is (n, n_levels+1) float64.  Replaces the diagonal pass of
 * sig_kernel_gram (kernels.py:589-595).  The symmetric Gram's diagonal
 * entries are formed from these values, so normalised diagonals are exactly 1.
 * FP32 paths (difference=1): level 1 is the exact telescoped sum of the
 * increments (kernels.py:281 summed: k(x_T,x_T) - 2k(x_0,x_T) + k(x_0,x_0),
 * float64); a sequence whose FP32 level 1 deviates from it by more than
 * 1e-5 relative, or with a negative or non-finite level, is recomputed in
 * float64.
 */
SK_API int sk_self_levels(const double *X, int64_t n, int64_t l, int64_t d,
                   const sk_kernel_config *cfg, double *out,
                   void *workspace, size_t workspace_bytes, void *stream);

/*
 * Signature-kernel Gram block (kernels.py:530-600, algorithm="dp").
 *
 *  FP32 certification: on the FP32 paths every K entry is certified in the
 *  kernel epilogue, and entries that are not are recomputed in float64 by a
 *  fix-up kernel in the same stream (the pair's levels and, when normalised,
 *  both self levels), so every returned entry meets the north-star tolerance
 *  (1e-5 relative normalised, 1e-4 unnormalised) or is float64. Level 1 is
 *  replaced by its exact telescoped value (difference=1). An entry is
 *  uncertified if it is non-finite, if its FP32 level 1 deviates from the
 *  exact one by more than 1e-5 of its scale (sqrt(k_1(x,x) k_1(y,y))
 *  normalised, sum_m |k_m(x,y)| otherwise), or if it is small against its
 *  scale: |K| < 0.05 (normalised: the unit diagonal) or |K| < 0.01 sum_m
 *  |k_m(x,y)| (unnormalised: cross-level cancellation). Thresholds are
 *  calibrated on seeded sweeps.
 *  X (nx, lx, d), Y (ny, ly, d). symmetric=1 means Y is X (K(X) in the
 *  reference, `Y=None`): only pairs with i <= j are evaluated and K[i,j] is
 *  mirrored into K[j,i] bit for bit (kernels.py:449-468); Y/ny/ly are ignored.
 *
 *  Rows [row_begin, row_end) of X are evaluated (multi-GPU row sharding):
 *   - cross (symmetric=0): K points at the storage of row `row_begin`;
 *     K[(i-row_begin)*ldk + j].
 *   - symmetric: K points at row 0 of the full (nx, nx) matrix; pairs
 *     (i, j>=i) with i in the row range are written at [i,j] and [j,i].
 *  levels (optional, may be NULL): per-pair level values, laid out like K but
 *   with (n_levels+1) float64 per entry (row stride ldk*(n_levels+1)).
 *  diag_x (nx, M+1) / diag_y (ny, M+1): self levels from sk_self_levels,
 *   required when normalization != SK_NORM_NONE. For SK_NORM_GLOBAL the
 *   caller has already rejected non-positive self kernels (kernels.py:519-527).
 *  K may be NULL if only `levels` is wanted.
 */
SK_API int sk_gram(const double *X, int64_t nx, int64_t lx,
            const double *Y, int64_t ny, int64_t ly, int64_t d,
            int32_t symmetric, const sk_kernel_config *cfg,
            int64_t row_begin, int64_t row_end,
            const double *diag_x, const double *diag_y,
            double *K, int64_t ldk, double *levels,
            void *workspace, size_t workspace_bytes, void *stream);

/*
 * Level values from given increment matrices (sig_levels_dp, kernels.py:144-201):
 *  A is (batch, t1, t2) float64, or (n_levels, batch, t1, t2) when
 *  per_level=1 (level m consumes A[m-1], kernels.py:129-141).
 *  out is (batch, n_levels+1) float64.  Float64 arithmetic.
 */
SK_API size_t sk_levels_dp_workspace_bytes(int64_t batch, int64_t t1, int64_t t2,
                                    int32_t n_levels, int32_t order);
SK_API int sk_levels_dp(const double *A, int64_t batch, int64_t t1, int64_t t2,
                 int32_t n_levels, int32_t order, int32_t per_level,
                 double *out, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Increment matrices (increment_tensor, kernels.py:263-281), float64:
 *  paired=0: all pairs, out (nx, ny, T1, T2); paired=1: nx == ny, out (nx, T1, T2),
 *  with T = l-1 when difference=1 (0 if l < 2) and T = l otherwise.
 */
SK_API int sk_increment_tensor(const double *X, int64_t nx, int64_t lx,
                        const double *Y, int64_t ny, int64_t ly, int64_t d,
                        int32_t paired, const sk_static_spec *spec, int32_t difference,
                        double *out, void *stream);

/*
 * Pairwise Euclidean distances of n points (float64, (n, d) row-major), upper
 * triangle i < j row by row: out has n*(n-1)/2 entries. Same formula as the
 * reference's _pairwise_sqdist + sqrt (static/kernels.py:108-114, 183-184):
 * sqrt(max(|x_i|^2 + |x_j|^2 - 2<x_i, x_j>, 0)). Used by median_heuristic
 * (static/kernels.py:165-187) to derive an RBF bandwidth.
 */
SK_API int sk_pairwise_dist(const double *X, int64_t n, int64_t d, double *out, void *stream);

/*
 * Untruncated signature kernel by the Goursat-PDE solve (algorithm="pde",
 * kernels.py:334-507): float64, one row-streamed pair per thread.
 *  K: like sk_gram (cross: rows [row_begin,row_end) at K[(i-row_begin)*ldk+j];
 *  symmetric: full matrix, upper triangle evaluated and mirrored).
 *  sk_pde_self: k(x_i, x_i) for global normalisation, out is (n,).
 *  With difference=1 every sequence needs L >= 2 (one increment).
 */
SK_API size_t sk_pde_workspace_bytes(int64_t npairs, int64_t ly, int32_t difference);
SK_API int sk_pde_gram(const double *X, int64_t nx, int64_t lx, const double *Y, int64_t ny,
                int64_t ly, int64_t d, int32_t symmetric, const sk_static_spec *spec,
                int32_t difference, int64_t row_begin, int64_t row_end, double *K, int64_t ldk,
                void *workspace, size_t workspace_bytes, void *stream);
SK_API int sk_pde_self(const double *X, int64_t n, int64_t l, int64_t d,
                const sk_static_spec *spec, int32_t difference, double *out,
                void *workspace, size_t workspace_bytes, void *stream);

/*
 * rfsf_exact_gram (features.py:446-475): exact Gram of a fitted rfsf_full
 * random-feature map via its finite-rank lift (_lifted_level_grams,
 * features.py:397-424). Level m of the dual DP uses the static kernel
 * <phi_m(x), phi_m(y)> of slot m's feature map, so the DP consumes one
 * increment matrix per level (kernels.py:129-141). Float64 throughout.
 */
enum sk_feature_kind { SK_FEAT_RFF = 0, SK_FEAT_RFF1D = 1, SK_FEAT_NYSTROEM = 2 };

/* A fitted static feature map (StaticFeatureState, static/features.py:56-66);
 * every pointer is device memory. */
typedef struct sk_feature_map {
  int32_t kind;            /* sk_feature_kind */
  int32_t reserved;        /* must be 0 */
  int64_t n_components;    /* D */
  int64_t out_dim;         /* 2D (rff), D (rff1d), kept eigenvalues (nystroem) */
  const double *weights;   /* (d, D) frequencies: rff, rff1d */
  const double *phases;    /* (D,) offsets: rff1d */
  const double *landmarks; /* (D, d) landmark rows: nystroem */
  const double *whiten;    /* (D, out_dim): nystroem */
  sk_static_spec base;     /* nystroem base kernel */
} sk_feature_map;

/*
 * transform_static_features (static/features.py:102-124): X is (npts, d);
 * feature row p is written at out[p*ld_out + 0 .. out_dim). The nystroem map
 * needs sk_static_features_workspace_bytes of workspace (0 for rff kinds).
 */
SK_API size_t sk_static_features_workspace_bytes(const sk_feature_map *map, int64_t npts);
SK_API int sk_static_features(const sk_feature_map *map, const double *X, int64_t npts,
                       int64_t d, double *out, int64_t ld_out,
                       void *workspace, size_t workspace_bytes, void *stream);

/*
 * Lifted level Grams. UX (nx, lx, width) / UY (ny, ly, width) hold every
 * slot's features concatenated along the last axis; slot m (level m+1) owns
 * channels [slot_offsets[m], slot_offsets[m+1]), m = 0..n_levels-1
 * (slot_offsets is HOST memory, n_levels+1 entries). `order` is the effective
 * order; K / levels / rows / symmetric / diag as in sk_gram, diag from
 * sk_lifted_self_levels (_lifted_self_levels, features.py:427-443) when
 * normalization is SK_NORM_LEVELWISE.
 */
SK_API size_t sk_lifted_workspace_bytes(int64_t npairs, int64_t ly, int32_t n_levels,
                                 int32_t order, int32_t difference);
/* Workspace with which sk_lifted_gram precomputes the slot Grams
 * <phi_m(x_i[r]), phi_m(y_j[c])> block by block (float64 tiled GEMM, up to
 * 4 GiB per block) instead of forming the inner products inside the DP; with
 * only sk_lifted_workspace_bytes(nx*ny, ...) it runs the on-the-fly kernel.
 * sk_lifted_self_levels likewise precomputes per-sequence slot Grams with
 * sk_lifted_gram_workspace_bytes(n, l, 1, l, ...) bytes of workspace. */
SK_API size_t sk_lifted_gram_workspace_bytes(int64_t nx, int64_t lx, int64_t ny, int64_t ly,
                                      int32_t n_levels, int32_t order, int32_t difference);
SK_API int sk_lifted_gram(const double *UX, int64_t nx, int64_t lx, const double *UY,
                   int64_t ny, int64_t ly, int64_t width, const int64_t *slot_offsets,
                   int32_t n_levels, int32_t order, int32_t difference,
                   int32_t normalization, int32_t symmetric, int64_t row_begin,
                   int64_t row_end, const double *diag_x, const double *diag_y, double *K,
                   int64_t ldk, double *levels, void *workspace, size_t workspace_bytes,
                   void *stream);
SK_API int sk_lifted_self_levels(const double *UX, int64_t n, int64_t l, int64_t width,
                          const int64_t *slot_offsets, int32_t n_levels, int32_t order,
                          int32_t difference, double *out, void *workspace,
                          size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SIGKERN_B200_H */
