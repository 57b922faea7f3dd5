"""Randomised parity sweep: seeded random KernelConfigs and shapes through the
public `sig_kernel_gram`, whatever path each one dispatches to (fused FP32,
GEMM-fed FP32, float64), against the float64 CPU oracle.

Tolerances are the north star's, elementwise PLAIN relative error: 1e-5
normalised and 1e-4 unnormalised for anything that touched an FP32 kernel (the
Gram or either self-level pass), 1e-9 when everything ran in float64 (Matern
kinds: 1e-6, sqrt of the norm-expansion distance near x = y). Only entries
below 1e-12 of the matrix's largest are judged absolutely, and an entry
so ill-conditioned that float64 itself cannot pin it (the reference's own
rounding, estimated as 1e-14 x the level values of |A| — the DP on the
absolute increments — exceeds 1e-1 x the tolerance: one-dimensional paths with
many levels cancel terms ~1e12 times larger than the result) is held to that
float64 bound instead. The FP32 paths meet
this through their certification: entries the FP32 arithmetic cannot vouch for
(cancelling level sums, noisy increments) are recomputed in float64 inside
sk_gram (include/sigkern_b200.h). Seeds >= 96 alternate in n_levels 7-8 on
short sequences, where the cancellation lives (tools/fuzz_more.py runs the
same generator over more seeds).
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
    if seed >= 96 and seed % 2 == 0:  # second half: many levels on short sequences
        M = int(r.integers(7, 9))
        lx, ly = int(r.integers(8, 40)), int(r.integers(8, 40))
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


@pytest.mark.parametrize("seed", range(400))
def test_random_config_matches_oracle(seed):
    kind, kw, M, order, norm, diff, d, lx, ly, sym = _case(seed)
    X = gen_brownian(5, lx, d, SeedStream(seed, ("x",))).data
    Y = None if sym else gen_brownian(4, ly, d, SeedStream(seed, ("y",))).data
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=order,
                       difference=diff, normalization=norm)
    paths = {execution_path(lx, lx if sym else ly, d, cfg)}
    if norm != "none":  # self levels of X and Y dispatch on their own shapes
        paths |= {execution_path(lx, lx, d, cfg), execution_path(ly, ly, d, cfg)}
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
    if paths == {"fp64"}:
        # Matern: sqrt of the norm-expansion squared distance amplifies the
        # summation-order rounding near x = y (reference and kernel alike;
        # measured up to 2.9e-7 at d = 20-33 over 1000 extra seeds)
        tol = 1e-6 if kind.startswith("matern") else 1e-9
    else:
        tol = 1e-4 if norm == "none" else 1e-5
    floor = np.maximum(1e-12 * np.abs(R).max(), 10 / tol * _f64_error(X, Y, kind, kw, M, order,
                                                                        diff, norm))
    err = float((np.abs(K - R) / np.maximum(np.abs(R), floor)).max()) if R.size else 0.0
    assert err <= tol, (paths, kind, kw, M, order, norm, diff, d, lx, ly, sym, err)


def _f64_error(X, Y, kind, kw, M, order, diff, norm):
    """Rounding scale of the reference's own float64 value of every entry: 1e-14 x
    the level values of the DP on |A| (each level a sum of |terms|), normalised
    like the entry (levelwise: by the self levels; global: by the self kernels)."""
    sp = O.static_params(kind, **kw)
    Yr = X if Y is None else Y
    p = max(1, min(order, M)) if M >= 1 else 1
    A = np.abs(O.increments(sp, X[:, None], Yr[None, :], diff))
    mag = O.levels_dp(A, M, p)[..., 1:]
    if norm == "none":
        return 1e-14 * mag.sum(-1)
    dx = O.self_levels(sp, X, M, p, diff)
    dy = O.self_levels(sp, Yr, M, p, diff)
    if norm == "levelwise":
        den = np.sqrt(np.abs(dx[:, None, 1:] * dy[None, :, 1:]))
        t = np.divide(mag, den, out=np.zeros_like(mag), where=den > 0)
        return 1e-14 * t.sum(-1) / (M + 1)
    sx, sy = np.abs(dx.sum(-1)), np.abs(dy.sum(-1))
    return 1e-14 * mag.sum(-1) / np.sqrt(np.maximum(np.outer(sx, sy), 1e-300))
