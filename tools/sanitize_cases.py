"""Small cases of every kernel path for compute-sanitizer runs (tools/gpu_sanitize.sh)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import (KernelConfig, SeedStream, StaticKernelSpec, gen_brownian,  # noqa: E402
                                   median_heuristic, sig_kernel_gram, sig_levels_dp)
from paper_2501_07145_b200.kernels import execution_path  # noqa: E402

X = gen_brownian(9, 40, 3, SeedStream(1)).data
Y = gen_brownian(7, 40, 3, SeedStream(2)).data
cases = [
    ("fused p1 rbf levelwise", X, Y, KernelConfig(n_levels=5, normalization="levelwise")),
    ("fused p1 symmetric", X, None, KernelConfig(n_levels=4, normalization="global")),
    ("fused geometric", X, Y, KernelConfig(n_levels=4, order=4)),
    ("fused multi-panel", gen_brownian(5, 300, 2, SeedStream(3)).data,
     gen_brownian(4, 300, 2, SeedStream(4)).data, KernelConfig(n_levels=3, normalization="levelwise")),
    ("gemm linear d=20", gen_brownian(5, 40, 20, SeedStream(5)).data,
     gen_brownian(4, 40, 20, SeedStream(6)).data, KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=3)),
    ("gemm rbf d=20 levelwise", gen_brownian(5, 40, 20, SeedStream(5)).data,
     gen_brownian(4, 40, 20, SeedStream(6)).data, KernelConfig(n_levels=3, normalization="levelwise")),
    ("fused order 2", X, Y, KernelConfig(n_levels=3, order=2)),
    ("fp64 generic", X, Y, KernelConfig(n_levels=6, order=5)),
    # round 2: polynomial and many-level low-order fused kernels, the
    # certification redo (wide batched: linear d = 40 cancels), the row-scan
    # float64 kernels (long rows: column state in shared memory)
    ("fused polynomial", X, Y, KernelConfig(static=StaticKernelSpec(kind="polynomial", degree=3),
                                            n_levels=4)),
    ("fused (6,2)", X, Y, KernelConfig(n_levels=6, order=2, normalization="levelwise")),
    ("gemm linear d=40 redo", gen_brownian(6, 48, 40, SeedStream(7)).data,
     gen_brownian(5, 48, 40, SeedStream(8)).data,
     KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=3)),
    ("fused rbf M=8 short", gen_brownian(6, 12, 2, SeedStream(10)).data,
     gen_brownian(5, 12, 2, SeedStream(11)).data, KernelConfig(n_levels=8, normalization="levelwise")),
    ("fused matern32 (4,2)", X, Y, KernelConfig(static=StaticKernelSpec(kind="matern32"),
                                                n_levels=4, order=2, normalization="levelwise")),
    ("fused rbf nodiff (3,2)", X, Y, KernelConfig(n_levels=3, order=2, difference=False)),
    ("gemm rbf d=20 (5,3)", gen_brownian(5, 40, 20, SeedStream(5)).data,
     gen_brownian(4, 40, 20, SeedStream(6)).data, KernelConfig(n_levels=5, order=3)),
]
fp64_cases = [
    ("fp64 row-scan long rows", gen_brownian(2, 600, 2, SeedStream(12)).data,
     gen_brownian(2, 600, 2, SeedStream(13)).data, KernelConfig(n_levels=4)),
    ("fp64 row-scan wide", gen_brownian(3, 40, 40, SeedStream(14)).data,
     gen_brownian(2, 40, 40, SeedStream(15)).data, KernelConfig(n_levels=3, normalization="levelwise")),
]
for name, A, B, cfg in cases:
    K = sig_kernel_gram(A, B, cfg=cfg)
    L = A.shape[1]
    print(f"{name:28s} path={execution_path(L, L, A.shape[2], cfg):6s} finite={bool(np.isfinite(K).all())}")
for name, A, B, cfg in fp64_cases:
    K = sig_kernel_gram(A, B, cfg=cfg, precision="fp64")
    print(f"{name:28s} finite={bool(np.isfinite(K).all())}")
print("levels_dp", sig_levels_dp(np.random.default_rng(0).standard_normal((3, 6, 5)), 3, order=2).shape)
print("median", median_heuristic(X.reshape(-1, 3)))

# float64 PDE kernel and rfsf_exact_gram's feature + lifted kernels
from paper_2501_07145_b200.features import (SigFeatureConfig, StaticFeatureSpec,  # noqa: E402
                                            fit_sig_features, rfsf_exact_gram)
Kp = sig_kernel_gram(X[:4, :12], Y[:3, :12], cfg=KernelConfig(normalization="global"), algorithm="pde")
print("pde", bool(np.isfinite(Kp).all()))
Kp = sig_kernel_gram(X[:3, :40], None, cfg=KernelConfig(), algorithm="pde")  # 2 nodes per lane
print("pde sym", bool(np.isfinite(Kp).all()))
fc = SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind="rff"), n_components=4,
                      projection=4, n_levels=3, order=1)  # warp-per-pair lifted DP
st = fit_sig_features(fc, X[:4, :12], SeedStream(9))
print("rfsf order 1", bool(np.isfinite(rfsf_exact_gram(st, X[:4, :12], Y[:3, :12], normalize=True)).all()))
for kind in ("rff", "nystroem"):
    fc = SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind=kind), n_components=4,
                          projection=4, n_levels=3, order=2)
    st = fit_sig_features(fc, X[:4, :12], SeedStream(9))
    print("rfsf", kind, bool(np.isfinite(rfsf_exact_gram(st, X[:4, :12], Y[:3, :12], normalize=True)).all()))
