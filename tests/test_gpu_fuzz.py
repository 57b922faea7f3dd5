"""Randomised parity sweep: seeded random KernelConfigs and shapes through the
public `sig_kernel_gram`, whatever path each one dispatches to (fused FP32,
GEMM-fed FP32, float64), against the float64 CPU oracle.

Tolerances are the north star's (1e-5 normalised, 1e-4 unnormalised; entries
that cancel to ~0 are judged against 1e-3 of the largest entry) for the FP32
paths and 1e-9 for the float64 path (Matern kinds: 1e-7, sqrt of the
norm-expansion distance near x = y).
"""

import numpy as np
import pytest

from oracle import sigkern_oracle as O
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian
from paper_2501_07145_b200.kernels import execution_path, sig_kernel_gram

pytestmark = pytest.mark.gpu

KINDS = ("rbf", "linear", "matern12", "matern32", "matern52", "rational_quadratic", "polynomial")


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    kind = KINDS[int(r.integers(0, len(KINDS)))] if r.random() < 0.6 else "rbf"
    M = int(r.integers(1, 9))
    order = int(r.integers(1, M + 1)) if r.random() < 0.4 else 1
    norm = ("none", "levelwise", "global")[int(r.integers(0, 3))]
    diff = bool(r.random() < 0.85)
    d = int((1, 2, 3, 5, 8, 13, 16, 20, 33)[int(r.integers(0, 9))])
    lx = int(r.integers(2, 70))
    ly = int(r.integers(2, 70)) if r.random() < 0.6 else lx
    sym = bool(r.random() < 0.3)
    kw = {}
    if kind in ("rbf", "matern12", "matern32", "matern52", "rational_quadratic"):
        kw["bandwidth"] = float(r.uniform(0.5, 2.0))
    if kind == "rational_quadratic":
        kw["alpha"] = float(r.uniform(0.5, 3.0))
    if kind in ("linear", "polynomial"):
        kw["scale"] = float(r.uniform(0.3, 1.5))
    if kind == "polynomial":
        kw["degree"] = int(r.integers(1, 4))
        kw["gamma"] = float(r.uniform(0.5, 1.5))
    return kind, kw, M, order, norm, diff, d, lx, ly, sym


@pytest.mark.parametrize("seed", range(48))
def test_random_config_matches_oracle(seed):
    kind, kw, M, order, norm, diff, d, lx, ly, sym = _case(seed)
    X = gen_brownian(5, lx, d, SeedStream(seed, ("x",))).data
    Y = None if sym else gen_brownian(4, ly, d, SeedStream(seed, ("y",))).data
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=order,
                       difference=diff, normalization=norm)
    path = execution_path(lx, lx if sym else ly, d, cfg)
    try:
        R = O.gram(X, Y, sp=O.static_params(kind, **kw), M=M, p=order, difference=diff,
                   normalization=norm)
    except ArithmeticError:  # global normalisation of a non-positive self kernel
        with pytest.raises(ArithmeticError):
            sig_kernel_gram(X, Y, cfg=cfg)
        return
    K = sig_kernel_gram(X, Y, cfg=cfg)
    assert K.shape == R.shape
    if sym:
        assert np.array_equal(K, K.T)
    scale = np.maximum(np.abs(R), 1e-3 * np.abs(R).max())
    err = float((np.abs(K - R) / scale).max())
    if path == "fp64":
        tol = 1e-7 if kind.startswith("matern") else 1e-9
    else:
        tol = 1e-4 if norm == "none" else 1e-5
    assert err <= tol, (path, kind, kw, M, order, norm, diff, d, lx, ly, sym, err)
