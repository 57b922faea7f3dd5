"""Parity of the CUDA path with the reference (golden vectors) and the CPU oracle.

Tolerances (north star): max elementwise relative error vs float64 <= 1e-5 for
normalised kernels, <= 1e-4 unnormalised, for the FP32 path; the float64 path
is held to the reference's own 1e-10.
"""

import numpy as np
import pytest
import torch

from conftest import oracle_static, pkg_config
from oracle import sigkern_oracle as O
from paper_2501_07145_b200 import (KernelConfig, SeedStream, StaticKernelSpec, gen_brownian,
                                   increment_tensor, sig_kernel_dp, sig_kernel_gram,
                                   sig_levels_dp,
                                   uses_fast_path)

pytestmark = pytest.mark.gpu

TOL_NORM, TOL_RAW = 1e-5, 1e-4


def _rel(K, R):
    K = np.asarray(K)
    R = np.asarray(R)
    err = np.abs(K - R) / np.maximum(np.abs(R), 1e-300)
    err[(K == 0) & (R == 0)] = 0.0
    return float(err.max()) if err.size else 0.0


def test_library_kernels_launch():
    X = gen_brownian(4, 10, 2, SeedStream(3)).data
    K = sig_kernel_gram(X, cfg=KernelConfig(n_levels=3))
    assert K.shape == (4, 4) and np.isfinite(K).all()


def test_golden_cases_fp64(gram_cases):
    for name, X, Y, c, K_ref in gram_cases:
        # every case incl. the BASELINE blocks (c4: d = 128 block products; c5: rows of
        # 2047 increments, column state in the scratch slice) on the float64 kernels
        K = sig_kernel_gram(X, Y, cfg=pkg_config(c), precision="fp64")
        assert K.shape == K_ref.shape, name
        # Matern kinds take sqrt of the norm-expansion squared distance, which
        # amplifies summation-order rounding near x = y (different from BLAS);
        # everything else is held to the reference's own 1e-10.
        rtol = 1e-8 if c["kind"].startswith("matern") else 1e-10
        assert np.allclose(K, K_ref, rtol=rtol, atol=1e-12), (name, _rel(K, K_ref))


def test_golden_cases_fp32(gram_cases):
    n_fast = 0
    for name, X, Y, c, K_ref in gram_cases:
        cfg = pkg_config(c)
        K = sig_kernel_gram(X, Y, cfg=cfg)
        ly = X.shape[1] if Y is None else Y.shape[1]
        n_fast += uses_fast_path(X.shape[1], ly, X.shape[2], cfg)
        tol = TOL_RAW if c["normalization"] == "none" else TOL_NORM
        # plain relative error; only entries below 1e-12 of the largest are absolute
        scale = np.maximum(np.abs(K_ref), 1e-12 * np.abs(K_ref).max())
        err = float((np.abs(K - K_ref) / scale).max())
        assert err <= tol, (name, err)
    assert n_fast >= 20  # the fused kernels really ran on most cases


@pytest.mark.parametrize("name", ["bench_c1", "bench_c2", "bench_c2n", "bench_c3", "bench_c3u",
                                  "bench_c4", "bench_c5", "bench_c5n"])
def test_bench_config_blocks(gram_cases, name):
    """BASELINE configs (sub-blocks) vs the reference at the north-star tolerances."""
    _, X, Y, c, K_ref = gram_cases.get(name)
    K = sig_kernel_gram(X, Y, cfg=pkg_config(c))
    tol = TOL_RAW if c["normalization"] == "none" else TOL_NORM
    assert _rel(K, K_ref) <= tol, _rel(K, K_ref)


def test_symmetric_bitwise_and_unit_diagonal():
    X = gen_brownian(40, 50, 3, SeedStream(1)).data
    for norm in ("levelwise", "global"):
        K = sig_kernel_gram(X, cfg=KernelConfig(n_levels=5, normalization=norm))
        assert np.array_equal(K, K.T)
        assert np.array_equal(np.diag(K), np.ones(40)), norm


def test_symmetric_equals_cross_entries():
    X = gen_brownian(20, 30, 4, SeedStream(9)).data
    cfg = KernelConfig(n_levels=4)
    Ks = sig_kernel_gram(X, cfg=cfg)
    Kc = sig_kernel_gram(X, X, cfg=cfg)
    iu = np.triu_indices(20, 1)
    assert np.array_equal(Ks[iu], Kc[iu])  # same roles (row = streamed x) on the upper triangle
    # K(X)'s diagonal is the summed self levels (K(X, diag=True)); K(X, X)'s is a Gram pair
    assert np.allclose(np.diag(Ks), np.diag(Kc), rtol=1e-6, atol=0)


def test_deterministic():
    X = gen_brownian(64, 64, 8, SeedStream(2)).data
    Y = gen_brownian(48, 64, 8, SeedStream(3)).data
    cfg = KernelConfig(n_levels=5, normalization="levelwise")
    assert np.array_equal(sig_kernel_gram(X, Y, cfg=cfg), sig_kernel_gram(X, Y, cfg=cfg))


def test_row_blocks_compose():
    from paper_2501_07145_b200.kernels import gram_block
    X = torch.from_numpy(gen_brownian(70, 40, 5, SeedStream(4)).data).cuda()
    Y = torch.from_numpy(gen_brownian(33, 40, 5, SeedStream(5)).data).cuda()
    cfg = KernelConfig(n_levels=4, normalization="levelwise")
    full, _ = gram_block(X, Y, cfg)
    parts = [gram_block(X, Y, cfg, r0, r1)[0] for r0, r1 in ((0, 23), (23, 50), (50, 70))]
    assert torch.equal(torch.cat(parts), full)
    Ks = torch.zeros((70, 70), dtype=torch.float64, device="cuda")
    for r0, r1 in ((0, 10), (10, 40), (40, 70)):
        gram_block(X, None, cfg, r0, r1, K=Ks)
    assert torch.equal(Ks, gram_block(X, None, cfg)[0])


def test_fp32_vs_fp64_c3_shapes():
    X = gen_brownian(12, 256, 16, SeedStream(1)).data
    Y = gen_brownian(10, 256, 16, SeedStream(2)).data
    for norm, tol in (("levelwise", TOL_NORM), ("none", TOL_RAW)):
        cfg = KernelConfig(n_levels=5, normalization=norm)
        assert uses_fast_path(256, 256, 16, cfg)
        K32 = sig_kernel_gram(X, Y, cfg=cfg)
        K64 = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
        assert _rel(K32, K64) <= tol


def test_ragged_lengths_and_short_sequences():
    X = gen_brownian(5, 33, 3, SeedStream(6)).data
    Y = gen_brownian(4, 70, 3, SeedStream(7)).data
    cfg = KernelConfig(n_levels=4, normalization="levelwise")
    R = O.gram(X, Y, M=4, p=1, normalization="levelwise")
    assert _rel(sig_kernel_gram(X, Y, cfg=cfg), R) <= TOL_NORM
    assert _rel(sig_kernel_gram(Y, X, cfg=cfg), R.T) <= TOL_NORM
    Z = np.random.default_rng(0).standard_normal((3, 1, 3))  # one point: no increments
    K = sig_kernel_gram(Z, X, cfg=KernelConfig(n_levels=3))
    assert np.array_equal(K, np.ones((3, 5)))


@pytest.mark.parametrize("lx,ly", [(300, 300), (260, 600), (600, 270), (64, 300), (65, 520)])
def test_multi_panel_lengths(lx, ly):
    """L_y > 256: sequential 256-column panels chained through the carry buffer."""
    X = gen_brownian(6, lx, 4, SeedStream(11)).data
    Y = gen_brownian(5, ly, 4, SeedStream(12)).data
    for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM)):
        cfg = KernelConfig(n_levels=6, normalization=norm)
        assert uses_fast_path(lx, ly, 4, cfg)
        R = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
        assert _rel(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (lx, ly, norm)


def test_multi_panel_symmetric_and_blocks():
    from paper_2501_07145_b200.kernels import gram_block
    X = gen_brownian(21, 520, 3, SeedStream(13)).data
    cfg = KernelConfig(n_levels=4, normalization="levelwise")
    K = sig_kernel_gram(X, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(21))
    Xt = torch.from_numpy(X).cuda()
    Y = torch.from_numpy(gen_brownian(9, 520, 3, SeedStream(14)).data).cuda()
    full, _ = gram_block(Xt, Y, cfg)
    parts = [gram_block(Xt, Y, cfg, r0, r1)[0] for r0, r1 in ((0, 5), (5, 21))]
    assert torch.equal(torch.cat(parts), full)


def test_levels_dp_golden(levels_golden):
    z = levels_golden
    for t in range(24):
        A = z[f"dp{t}__A"]
        M, p = (int(v) for v in z[f"dp{t}__Mp"])
        assert np.allclose(sig_levels_dp(A, M, order=p), z[f"dp{t}__dp"], rtol=1e-10, atol=1e-12)
    mats = list(z["perlevel__A"])
    assert np.allclose(sig_levels_dp(mats, 3, order=2), z["perlevel__dp"], rtol=1e-10)
    assert np.allclose(sig_levels_dp(z["batched__A"], 4, order=2), z["batched__dp"], rtol=1e-10)


def test_increment_tensor_golden(levels_golden):
    z = levels_golden
    for kind in O.KINDS:
        spec = StaticKernelSpec(kind=kind, bandwidth=1.2)
        x, y = z[f"inc_{kind}__x"], z[f"inc_{kind}__y"]
        assert np.allclose(increment_tensor(spec, x, y), z[f"inc_{kind}__A"], atol=1e-12)
        assert np.allclose(increment_tensor(spec, x, y, difference=False), z[f"inc_{kind}__G"],
                           atol=1e-12)


def test_torch_tensors_stay_on_device():
    X = torch.from_numpy(gen_brownian(8, 20, 3, SeedStream(8)).data).cuda()
    K = sig_kernel_gram(X, cfg=KernelConfig(n_levels=3, normalization="levelwise"))
    assert isinstance(K, torch.Tensor) and K.is_cuda and K.shape == (8, 8)


def test_full_c3_prefix_block(gram_cases):
    """Full-size c3 cross Gram is out of the oracle's reach; its top-left block
    must equal the golden 4x4 block (inputs are prefix-stable), and all
    entries of a normalised Gram lie in [-1, 1] up to rounding."""
    _, X4, Y4, c, K_ref = gram_cases.get("bench_c3")
    n = 1024
    X = gen_brownian(n, 256, 16, SeedStream(1)).data
    Y = gen_brownian(n, 256, 16, SeedStream(2)).data
    assert np.array_equal(X[:4], X4) and np.array_equal(Y[:4], Y4)
    K = sig_kernel_gram(X, Y, cfg=pkg_config(c))
    assert _rel(K[:4, :4], K_ref) <= TOL_NORM
    assert np.isfinite(K).all() and np.abs(K).max() <= 1.0 + 1e-6


def _scaled_err(K, R):
    """Plain relative error; only entries below 1e-12 of the largest are judged absolutely."""
    K, R = np.asarray(K), np.asarray(R)
    scale = np.maximum(np.abs(R), 1e-12 * np.abs(R).max())
    return float((np.abs(K - R) / scale).max())


@pytest.mark.parametrize("M", [2, 3, 4, 5])
@pytest.mark.parametrize("kind", ["rbf", "linear"])
def test_geometric_order_fused(M, kind):
    """order = n_levels (geometric) runs on the fused FP32 kernel (kernels.py:179-199)."""
    X = gen_brownian(7, 60, 5, SeedStream(21)).data
    Y = gen_brownian(6, 45, 5, SeedStream(22)).data
    sp = O.static_params(kind)
    for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM)):
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=M, order=M,
                           normalization=norm)
        fused = not (kind == "linear" and norm != "none")  # see plan_for (sk_fast.cu)
        assert uses_fast_path(60, 45, 5, cfg) == fused and uses_fast_path(45, 60, 5, cfg) == fused
        if not fused:
            tol = 1e-10
        R = O.gram(X, Y, sp=sp, M=M, p=M, normalization=norm)
        assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (M, kind, norm)
        assert _scaled_err(sig_kernel_gram(Y, X, cfg=cfg), R.T) <= tol, (M, kind, norm)


def test_geometric_multi_panel_symmetric():
    """L > 128: the general-order kernel's 128-column panels chained through the carry."""
    X = gen_brownian(9, 300, 3, SeedStream(23)).data
    Y = gen_brownian(5, 140, 3, SeedStream(24)).data
    for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM)):
        cfg = KernelConfig(n_levels=4, order=4, normalization=norm)
        assert uses_fast_path(300, 300, 3, cfg)
        R = O.gram(X, Y, M=4, p=4, normalization=norm)
        assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, norm
        assert _scaled_err(sig_kernel_gram(Y, X, cfg=cfg), R.T) <= tol, norm
    cfg = KernelConfig(n_levels=5, order=5, normalization="levelwise")
    K = sig_kernel_gram(X, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(9))
    assert _scaled_err(K, O.gram(X, None, M=5, p=5, normalization="levelwise")) <= TOL_NORM


def test_c2_shapes_fused_vs_fp64():
    """c2 (L=128, d=8, M=p=5) sub-block: fused FP32 geometric kernel vs the float64 kernel."""
    X = gen_brownian(10, 128, 8, SeedStream(1)).data
    Y = gen_brownian(9, 128, 8, SeedStream(2)).data
    for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM)):
        cfg = KernelConfig(n_levels=5, order=5, normalization=norm)
        assert uses_fast_path(128, 128, 8, cfg)
        K32 = sig_kernel_gram(X, Y, cfg=cfg)
        K64 = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
        assert _rel(K32, K64) <= tol, norm


# ---------------------------------------------------------------------------
# GEMM-fed path (d > 16 or long x): library GEMM of the cell values + FP32 DP
# ---------------------------------------------------------------------------

def test_gemm_path_linear_c4_shapes():
    """c4 shapes (linear, d=128, M=3, unnormalised) sub-block vs the oracle."""
    from paper_2501_07145_b200.kernels import execution_path
    X = gen_brownian(6, 128, 128, SeedStream(1)).data
    Y = gen_brownian(5, 128, 128, SeedStream(2)).data
    cfg = KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=3)
    assert execution_path(128, 128, 128, cfg) == "gemm"
    R = O.gram(X, Y, sp=O.static_params("linear"), M=3, p=1)
    assert _rel(sig_kernel_gram(X, Y, cfg=cfg), R) <= TOL_RAW


@pytest.mark.parametrize("kind", ["rbf", "linear"])
@pytest.mark.parametrize("M,p", [(4, 1), (3, 3), (4, 2), (5, 3), (8, 2)])
def test_gemm_path_kinds_orders(kind, M, p):
    """d = 24: linear on the GEMM-fed path at every order; rbf on the float64
    kernel (its tensor-core cell values cannot hold the bar)."""
    from paper_2501_07145_b200.kernels import execution_path
    X = gen_brownian(7, 70, 24, SeedStream(31)).data
    Y = gen_brownian(6, 50, 24, SeedStream(32)).data
    sp = O.static_params(kind)
    norms = (("none", TOL_RAW),) if (kind == "linear" and p > 1) else \
        (("none", TOL_RAW), ("levelwise", TOL_NORM))
    for norm, tol in norms:
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=M, order=p,
                           normalization=norm)
        assert execution_path(70, 50, 24, cfg) == ("gemm" if kind == "linear" else "fp64")
        R = O.gram(X, Y, sp=sp, M=M, p=p, normalization=norm)
        assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (kind, M, p, norm)
        assert _scaled_err(sig_kernel_gram(Y, X, cfg=cfg), R.T) <= tol, (kind, M, p, norm)


def test_gemm_path_multi_panel_symmetric_blocks():
    from paper_2501_07145_b200.kernels import gram_block
    X = gen_brownian(9, 300, 20, SeedStream(33)).data
    cfg = KernelConfig(n_levels=4, normalization="levelwise")
    K = sig_kernel_gram(X, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(9))
    assert _rel(K, O.gram(X, None, M=4, p=1, normalization="levelwise")) <= TOL_NORM
    Xt = torch.from_numpy(X).cuda()
    Yt = torch.from_numpy(gen_brownian(4, 280, 20, SeedStream(34)).data).cuda()
    full, _ = gram_block(Xt, Yt, cfg)
    parts = [gram_block(Xt, Yt, cfg, r0, r1)[0] for r0, r1 in ((0, 4), (4, 9))]
    assert torch.equal(torch.cat(parts), full)


# ---------------------------------------------------------------------------
# tcgen05 3xTF32 GEMM (cell-value stage of the GEMM-fed path)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("M,N,K", [(128, 256, 32), (300, 520, 132), (1000, 77, 128)])
def test_tc_gemm_3xtf32_matches_fp64(M, N, K):
    import ctypes
    from paper_2501_07145_b200 import _native
    lib = _native.load()
    g = torch.Generator(device="cpu").manual_seed(M + N + K)
    A = torch.randn(M, K, generator=g, dtype=torch.float64)
    B = torch.randn(N, K, generator=g, dtype=torch.float64)
    A32, B32 = A.float().cuda(), B.float().cuda()
    ldc = M + 3
    C = torch.full((N, ldc), float("nan"), dtype=torch.float32, device="cuda")
    scratch = torch.empty(2 * (M + N) * K, dtype=torch.float32, device="cuda")
    fn = lib.sk_dev_tc_gemm
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    rc = fn(A32.data_ptr(), M, B32.data_ptr(), N, K, C.data_ptr(), ldc, scratch.data_ptr(),
            torch.cuda.current_stream().cuda_stream)
    assert rc == 0, lib.sk_last_error()
    torch.cuda.synchronize()
    ref = (B32.double() @ A32.double().T).cpu()  # exact products of the fp32 inputs
    got = C[:, :M].double().cpu()
    scale = (B32.double().abs() @ A32.double().abs().T).cpu()
    err = float(((got - ref).abs() / scale).max())
    assert err < 1e-6, err  # 3xTF32 ~ FP32 accuracy (1xTF32 would be ~1e-3)
    assert torch.isnan(C[:, M:]).all()  # nothing written beyond the M columns


def test_median_heuristic_golden():
    """median_heuristic (static/kernels.py:165-187) vs the reference's own values."""
    import os
    from paper_2501_07145_b200 import median_heuristic
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "median.npz"))
    names = sorted({k.split("__")[0] for k in z.files})
    for name in names:
        got = median_heuristic(z[f"{name}__X"], max_pairs=int(z[f"{name}__max_pairs"]))
        assert got == pytest.approx(float(z[f"{name}__median"]), rel=1e-12), name
    assert median_heuristic(np.zeros((4, 2))) == 1.0
    with pytest.raises(ValueError, match="at least 2"):
        median_heuristic(np.zeros((1, 2)))
    with pytest.raises(ValueError, match="max_pairs"):
        median_heuristic(np.zeros((3, 2)), max_pairs=0)


# ---------------------------------------------------------------------------
# the reference's own known-answer tests, re-pointed at the device path
# ---------------------------------------------------------------------------

LIN = StaticKernelSpec(kind="linear")


def test_criterion_01_device_dp_matches_bruteforce():
    """test_acceptance.py:61-87: 200 random instances, L <= 5, d <= 3, M <= 3,
    p in {1, 2}; float64 path at 1e-10, FP32 paths at the north-star 1e-4."""
    rng = np.random.default_rng(20240601)
    worst64 = worst32 = 0.0
    for _ in range(200):
        L1, L2 = rng.integers(2, 6, size=2)
        d = int(rng.integers(1, 4))
        M = int(rng.integers(0, 4))
        p = int(rng.integers(1, 3))
        bw = float(rng.uniform(0.5, 2.0))
        static = LIN if rng.integers(2) == 0 else StaticKernelSpec(kind="rbf", bandwidth=bw)
        cfg = KernelConfig(static=static, n_levels=M, order=p)
        x = rng.standard_normal((L1, d))
        y = rng.standard_normal((L2, d))
        sp = O.static_params(static.kind, bandwidth=static.bandwidth)
        bf = O.levels_bruteforce(O.increments(sp, x, y), M, cfg.effective_order)
        for prec in ("fp64", "fp32"):
            dp = np.asarray(sig_kernel_dp(x, y, cfg, precision=prec).values)
            rel = np.abs(dp - bf) / np.maximum(np.abs(bf), 1e-30)
            rel[(dp == 0.0) & (bf == 0.0)] = 0.0
            # FP32: judge near-cancelling levels against the level-1 scale
            sc = np.maximum(np.abs(bf), 1e-3 * max(1.0, float(np.abs(bf).max())))
            if prec == "fp64":
                worst64 = max(worst64, float(rel.max()))
            else:
                worst32 = max(worst32, float((np.abs(dp - bf) / sc).max()))
    assert worst64 <= 1e-10, worst64
    assert worst32 <= TOL_RAW, worst32


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_criterion_02_hand_values(prec):
    """test_acceptance.py:90-100: linear, x increments (1, 2), y increment (2):
    k_1 = 6; k_2 = 0 at p = 1, 9 at p = 2."""
    x = np.array([[0.0], [1.0], [3.0]])
    y = np.array([[0.0], [2.0]])
    lv1 = sig_kernel_dp(x, y, KernelConfig(static=LIN, n_levels=2, order=1), precision=prec)
    lv2 = sig_kernel_dp(x, y, KernelConfig(static=LIN, n_levels=2, order=2), precision=prec)
    assert abs(lv1[1] - 6.0) <= 1e-12 and lv1[2] == 0.0 and abs(lv2[2] - 9.0) <= 1e-12


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_constant_sequences_give_unit_level_zero(prec):
    """test_kernels.py:67-72: constant sequences -> (1, 0, ..., 0) exactly."""
    x = np.ones((4, 2)) * 0.3
    y = np.ones((3, 2)) * -1.0
    for cfg in (KernelConfig(static=LIN, n_levels=4, order=2), KernelConfig(n_levels=4),
                KernelConfig(n_levels=4, order=4)):
        assert np.array_equal(np.asarray(sig_kernel_dp(x, y, cfg, precision=prec).values),
                              [1.0, 0, 0, 0, 0])


def test_normalised_gram_is_psd_on_fused_paths():
    """test_kernels.py:428-433: normalised K(X) is positive semi-definite."""
    X = gen_brownian(30, 40, 3, SeedStream(41)).data
    for cfg in (KernelConfig(n_levels=5, normalization="levelwise"),
                KernelConfig(n_levels=4, order=4, normalization="levelwise"),
                KernelConfig(n_levels=3, normalization="global")):
        assert uses_fast_path(40, 40, 3, cfg)
        K = sig_kernel_gram(X, cfg=cfg)
        assert np.linalg.eigvalsh(K).min() >= -1e-6


# ---------------------------------------------------------------------------
# algorithm="pde" (kernels.py:334-507): float64 Goursat solve on the device
# ---------------------------------------------------------------------------

def test_pde_golden_gram():
    from test_oracle_golden import _pde_cases
    for name, X, Y, sp, diff, norm, K_ref, kind, par in _pde_cases():
        spec = StaticKernelSpec(kind=kind, **({"scale": par} if kind == "linear" else {"bandwidth": par}))
        cfg = KernelConfig(static=spec, difference=diff, normalization=norm)
        K = sig_kernel_gram(X, Y, cfg=cfg, algorithm="pde")
        assert K.shape == K_ref.shape
        assert np.allclose(K, K_ref, rtol=1e-11, atol=0), (name, _rel(K, K_ref))
        if Y is None:
            assert np.array_equal(K, K.T)


@pytest.mark.parametrize("lx,ly,d,kind,diff", [
    (5, 7, 3, "rbf", True), (40, 33, 2, "linear", True), (70, 100, 5, "rbf", True),
    (150, 200, 3, "matern32", True), (12, 9, 20, "rbf", True), (30, 140, 12, "rbf", False),
    (300, 280, 2, "rbf", True)])
def test_pde_shapes_vs_oracle(lx, ly, d, kind, diff):
    """Warp-per-pair systolic solve (columns per lane 1..8, registers or memory
    for the points) and the long-sequence thread-per-pair fallback, vs the oracle."""
    X = gen_brownian(3, lx, d, SeedStream(81)).data
    Y = gen_brownian(2, ly, d, SeedStream(82)).data
    kw = {"scale": 0.8} if kind == "linear" else {"bandwidth": 1.1}
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), difference=diff)
    sp = O.static_params(kind, **kw)
    K = sig_kernel_gram(X, Y, cfg=cfg, algorithm="pde")
    rtol = 1e-8 if kind.startswith("matern") else 1e-11
    assert np.allclose(K, O.pde_gram(X, Y, sp=sp, difference=diff), rtol=rtol, atol=0)
    Ks = sig_kernel_gram(X, cfg=cfg, algorithm="pde")
    assert np.array_equal(Ks, Ks.T)
    assert np.allclose(Ks, O.pde_gram(X, None, sp=sp, difference=diff), rtol=rtol, atol=0)


def test_pde_hand_values_and_errors():
    """test_kernels.py:233-262 re-pointed at the device path."""
    from paper_2501_07145_b200 import sig_pde_kernel
    x = np.ones((3, 2))
    assert sig_pde_kernel(x, x, KernelConfig(static=LIN)) == 1.0
    x = np.array([[0.0], [1.0]])
    assert sig_pde_kernel(x, x, KernelConfig(static=LIN)) == pytest.approx(2.0)
    with pytest.raises(ValueError, match="increment"):
        sig_pde_kernel(np.array([[1.0]]), np.array([[1.0]]), KernelConfig(static=LIN))
    one = np.array([[1.0]])
    assert sig_pde_kernel(one, one, KernelConfig(static=LIN, difference=False)) == pytest.approx(2.0)


def test_pde_second_order_convergence():
    """test_acceptance.py:103-125: dyadic refinement of the unit linear path converges
    to sum 1/(m!)^2 with error ratios in [3, 6]."""
    import math
    from paper_2501_07145_b200 import sig_pde_kernel
    target = sum(1.0 / math.factorial(m) ** 2 for m in range(30))
    errs = []
    for r in range(9):
        path = np.linspace(0.0, 1.0, 2 ** r + 1)[:, None]
        errs.append(abs(sig_pde_kernel(path, path, KernelConfig(static=LIN)) - target))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    assert all(3.0 <= q <= 6.0 for q in ratios[2:]), ratios


def test_pde_vs_truncated_consistency():
    """test_acceptance.py:128-145: PDE ~ truncated M=10, p=5 kernel at small increments."""
    from paper_2501_07145_b200 import sig_pde_kernel
    cfg = KernelConfig(static=StaticKernelSpec(kind="rbf", bandwidth=2.0), n_levels=10, order=5)
    rng = np.random.default_rng(0)
    worst = 0.0
    for _ in range(10):
        X = np.vstack([np.zeros((1, 2)), np.cumsum(0.1 * rng.standard_normal((5, 2)), axis=0)])
        Y = np.vstack([np.zeros((1, 2)), np.cumsum(0.1 * rng.standard_normal((5, 2)), axis=0)])
        pde = sig_pde_kernel(X, Y, cfg)
        dp = sig_kernel_dp(X, Y, cfg, precision="fp64").total()
        worst = max(worst, abs(pde - dp) / abs(pde))
    assert worst <= 1e-3, worst


# ---------------------------------------------------------------------------
# CUDA-graph plans (plan.GramPlan / SignatureKernel(cuda_graph=True))
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("norm", ["levelwise", "none", "global"])
def test_graph_plan_matches_eager_bitwise(norm):
    import time
    from paper_2501_07145_b200 import RBFKernel, SignatureKernel
    X = gen_brownian(64, 50, 3, SeedStream(1)).data
    Y = gen_brownian(48, 50, 3, SeedStream(2)).data
    eager = SignatureKernel(n_levels=5, normalization=norm, static_kernel=RBFKernel(),
                            cuda_graph=False)
    graph = SignatureKernel(n_levels=5, normalization=norm, static_kernel=RBFKernel(),
                            cuda_graph=True)
    for A, B in ((X, None), (X, Y)):
        want = eager(A, B)
        assert np.array_equal(graph(A, B), want)
        A2 = A + 0.01  # same plan, new inputs
        assert np.array_equal(graph(A2, B), eager(A2, B))
    Xt = torch.from_numpy(X).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        Kg = graph(Xt)
    torch.cuda.synchronize()
    tg = (time.perf_counter() - t0) / 50
    t0 = time.perf_counter()
    for _ in range(50):
        Ke = eager(Xt)
    torch.cuda.synchronize()
    te = (time.perf_counter() - t0) / 50
    assert torch.equal(Kg, Ke)
    print(f"c1 K(X) {norm}: graph {1e6 * tg:.0f} us/call, eager {1e6 * te:.0f} us/call")


@pytest.mark.parametrize("kind", ["linear"])
def test_graph_plan_gemm_path_bitwise(kind):
    """CUDA-graph capture of the GEMM-fed path: cluster launches of the 2-SM
    tcgen05 GEMM (cudaLaunchKernelEx) and the DP replay bitwise."""
    from paper_2501_07145_b200 import LinearKernel, RBFKernel, SignatureKernel
    from paper_2501_07145_b200.kernels import execution_path
    X = gen_brownian(9, 40, 24, SeedStream(5)).data
    Y = gen_brownian(7, 40, 24, SeedStream(6)).data
    static = LinearKernel() if kind == "linear" else RBFKernel()
    norm = "none" if kind == "linear" else "levelwise"
    eager = SignatureKernel(n_levels=3, normalization=norm, static_kernel=static, cuda_graph=False)
    graph = SignatureKernel(n_levels=3, normalization=norm, static_kernel=static, cuda_graph=True)
    assert execution_path(40, 40, 24, eager.config if hasattr(eager, "config") else
                          KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=3,
                                       normalization=norm)) == "gemm"
    for A, B in ((X, Y), (X, None), (X + 0.02, Y)):
        assert np.array_equal(graph(A, B), eager(A, B))


def test_facade_auto_graph_for_launch_bound_calls():
    """cuda_graph='auto' (the default): small Grams replay a captured plan, bitwise
    equal to the eager call; large ones, other devices' tensors and SequenceBatch
    inputs stay eager; errors keep the eager messages."""
    from paper_2501_07145_b200 import RBFKernel, SignatureKernel
    auto = SignatureKernel(n_levels=5, static_kernel=RBFKernel())
    eager = SignatureKernel(n_levels=5, static_kernel=RBFKernel(), cuda_graph=False)
    X = gen_brownian(64, 50, 3, SeedStream(21)).data
    Xt = torch.from_numpy(X).cuda()
    assert np.array_equal(auto(X), eager(X))
    assert torch.equal(auto(Xt), eager(Xt))
    assert len(auto._plans) == 1  # one plan per shape, numpy or tensor inputs
    big = torch.zeros((1024, 256, 3), dtype=torch.float64, device="cuda")
    assert not auto._use_graph(big, None)
    assert not auto._use_graph(np.zeros((4, 1, 3)), None)  # no increments
    bad = X.copy()
    bad[1, 3, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        auto(bad)
    with pytest.raises(ValueError):
        SignatureKernel(cuda_graph="sometimes")


def test_graph_plan_errors():
    from paper_2501_07145_b200.plan import GramPlan
    plan = GramPlan(KernelConfig(n_levels=3, normalization="global"), (4, 10, 2))
    X = gen_brownian(4, 10, 2, SeedStream(3)).data
    plan(X)
    bad = X.copy()
    bad[1, 3, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        plan(bad)
    with pytest.raises(ValueError, match="shape"):
        plan(X[:3])
    const = np.zeros((4, 10, 2))  # zero self-kernels beyond level 0 are fine (level 0 = 1)
    plan(const)


# ---------------------------------------------------------------------------
# stationary static kinds on the fused FP32 kernel (StatPointStage)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kind", ["matern12", "matern32", "matern52", "rational_quadratic"])
def test_stationary_kinds_fused(kind):
    X = gen_brownian(7, 60, 5, SeedStream(51)).data
    Y = gen_brownian(6, 45, 5, SeedStream(52)).data
    extra = dict(alpha=1.7) if kind == "rational_quadratic" else {}
    spec = StaticKernelSpec(kind=kind, bandwidth=0.9, **extra)
    sp = O.static_params(kind, bandwidth=0.9, **extra)
    for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM), ("global", TOL_NORM)):
        cfg = KernelConfig(static=spec, n_levels=5, normalization=norm)
        assert uses_fast_path(60, 45, 5, cfg)
        R = O.gram(X, Y, sp=sp, M=5, p=1, normalization=norm)
        assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (kind, norm)
    cfg = KernelConfig(static=spec, n_levels=4, normalization="levelwise")
    K = sig_kernel_gram(X, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(7))
    assert _scaled_err(K, O.gram(X, None, sp=sp, M=4, p=1, normalization="levelwise")) <= TOL_NORM


@pytest.mark.parametrize("kind,M,p", [("matern12", 3, 2), ("matern32", 4, 4), ("matern52", 5, 3),
                                      ("rational_quadratic", 5, 5), ("matern32", 8, 2)])
def test_stationary_kinds_general_order_fused(kind, M, p):
    """Matern / rational quadratic at 1 < p <= M on the general-order fused kernel."""
    X = gen_brownian(6, 50, 5, SeedStream(55)).data
    Y = gen_brownian(5, 41, 5, SeedStream(56)).data
    extra = dict(alpha=1.3) if kind == "rational_quadratic" else {}
    spec = StaticKernelSpec(kind=kind, bandwidth=1.1, **extra)
    sp = O.static_params(kind, bandwidth=1.1, **extra)
    for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM)):
        cfg = KernelConfig(static=spec, n_levels=M, order=p, normalization=norm)
        assert uses_fast_path(50, 41, 5, cfg)
        R = O.gram(X, Y, sp=sp, M=M, p=p, normalization=norm)
        assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (kind, norm)
    cfg = KernelConfig(static=spec, n_levels=M, order=p, normalization="levelwise")
    Xl = gen_brownian(3, 300, 3, SeedStream(57)).data  # multi-panel, symmetric
    K = sig_kernel_gram(Xl, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(3))
    assert _scaled_err(K, O.gram(Xl, None, sp=sp, M=M, p=p, normalization="levelwise")) <= TOL_NORM


def test_stationary_kind_multi_panel():
    X = gen_brownian(4, 300, 3, SeedStream(53)).data
    Y = gen_brownian(3, 280, 3, SeedStream(54)).data
    spec = StaticKernelSpec(kind="matern32", bandwidth=1.2)
    cfg = KernelConfig(static=spec, n_levels=4, normalization="levelwise")
    assert uses_fast_path(300, 280, 3, cfg)
    R = O.gram(X, Y, sp=O.static_params("matern32", bandwidth=1.2), M=4, p=1,
               normalization="levelwise")
    assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= TOL_NORM


@pytest.mark.parametrize("degree,gamma", [(1, 0.5), (2, 1.0), (3, 1.3)])
def test_polynomial_float64(degree, gamma):
    """Polynomial kind (static/kernels.py:68-71) runs on the float64 kernels: its
    FP32 recursion loses to cancellation inside the high levels, which the
    certification cannot see. Single and long rows, every
    normalisation, general order, symmetric."""
    from paper_2501_07145_b200.kernels import execution_path
    spec = StaticKernelSpec(kind="polynomial", scale=0.7, degree=degree, gamma=gamma)
    sp = O.static_params("polynomial", scale=0.7, degree=degree, gamma=gamma)
    for lx, ly, M, p in ((60, 45, 4, 1), (300, 270, 3, 1), (45, 38, 4, 2)):
        X = gen_brownian(4, lx, 6, SeedStream(71)).data
        Y = gen_brownian(3, ly, 6, SeedStream(72)).data
        for norm in ("none", "levelwise", "global"):
            cfg = KernelConfig(static=spec, n_levels=M, order=p, normalization=norm)
            assert execution_path(lx, ly, 6, cfg) == "fp64"
            try:
                R = O.gram(X, Y, sp=sp, M=M, p=p, normalization=norm)
            except ArithmeticError:
                continue
            err = _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R)
            assert err <= 1e-9, (degree, lx, norm, err)
    X = gen_brownian(5, 50, 6, SeedStream(73)).data
    cfg = KernelConfig(static=spec, n_levels=5, normalization="levelwise")
    K = sig_kernel_gram(X, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(5))
    assert _scaled_err(K, O.gram(X, None, sp=sp, M=5, p=1, normalization="levelwise")) <= 1e-9


@pytest.mark.parametrize("kind", ["rbf", "linear"])
def test_difference_false_fused(kind):
    """difference=False (kernels.py:275-276): A = G on the L x L' grid, fused FP32."""
    X = gen_brownian(6, 40, 3, SeedStream(61)).data
    Y = gen_brownian(5, 33, 3, SeedStream(62)).data
    sp = O.static_params(kind)
    orders = (1, 3) if kind == "linear" else (1, 2, 3)
    for p in orders:
        for norm, tol in (("none", TOL_RAW), ("levelwise", TOL_NORM)):
            if kind == "linear" and p > 1 and norm != "none":
                continue
            cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=3, order=p,
                               difference=False, normalization=norm)
            assert uses_fast_path(40, 33, 3, cfg)
            R = O.gram(X, Y, sp=sp, M=3, p=p, difference=False, normalization=norm)
            assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (kind, p, norm)
            assert _scaled_err(sig_kernel_gram(Y, X, cfg=cfg), R.T) <= tol, (kind, p, norm)
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=3, difference=False,
                       normalization="levelwise")
    K = sig_kernel_gram(X, cfg=cfg)
    assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(6))
    one = np.random.default_rng(3).standard_normal((2, 1, 3))  # one point = one raw cell
    R1 = O.gram(one, one, sp=sp, M=3, p=1, difference=False)
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=3, difference=False)
    assert _scaled_err(sig_kernel_gram(one, one, cfg=cfg), R1) <= TOL_RAW


# ---------------------------------------------------------------------------
# full BASELINE sizes: the whole Gram on the device, checked through its
# prefix-stable golden block (gen_brownian is prefix-stable: the first k
# sequences of the full batch are the golden inputs) and size-independent
# properties
# ---------------------------------------------------------------------------

FULL = {  # name: (N, L, d, golden case)
    "c3": (8192, 256, 16, "bench_c3"),
    "c3u": (8192, 256, 16, "bench_c3u"),
    "c2": (1024, 128, 8, "bench_c2"),
    "c2n": (1024, 128, 8, "bench_c2n"),
    "c4": (4096, 128, 128, "bench_c4"),
    "c5": (512, 2048, 4, "bench_c5"),
    "c5n": (512, 2048, 4, "bench_c5n"),
}


@pytest.mark.parametrize("name", sorted(FULL))
def test_full_size_baseline_configs(gram_cases, name):
    N, L, d, golden = FULL[name]
    _, Xg, Yg, c, K_ref = gram_cases.get(golden)
    k = Xg.shape[0]
    X = torch.from_numpy(gen_brownian(N, L, d, SeedStream(1)).data).cuda()
    Y = torch.from_numpy(gen_brownian(N, L, d, SeedStream(2)).data).cuda()
    assert np.array_equal(X[:k].cpu().numpy(), Xg) and np.array_equal(Y[:k].cpu().numpy(), Yg)
    cfg = pkg_config(c)
    K = sig_kernel_gram(X, Y, cfg=cfg)
    assert K.shape == (N, N) and bool(torch.isfinite(K).all())
    tol = TOL_RAW if c["normalization"] == "none" else TOL_NORM
    assert _rel(K[:k, :k].cpu().numpy(), K_ref) <= tol
    if c["normalization"] != "none":
        assert float(K.abs().max()) <= 1.0 + 1e-6
    if name in ("c3", "c3u"):
        # the far-end 24 x 24 block against the reference (tests/golden/c3_far.npz)
        import os
        z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c3_far.npz"))
        far = K[N - 24:, N - 24:].cpu().numpy()
        assert _rel(far, z["K_levelwise" if name == "c3" else "K_none"]) <= tol
    # row blocks of the full Gram are the Gram of the row blocks (no cross-row state)
    rows = torch.arange(N - 3, N, device="cuda")
    Kb = sig_kernel_gram(X[rows], Y, cfg=cfg)
    assert torch.equal(Kb, K[rows])


@pytest.mark.parametrize("M,p", [(3, 2), (4, 2), (4, 3), (5, 2), (5, 3), (5, 4),
                                 (6, 2), (6, 3), (7, 2), (8, 2)])
def test_intermediate_orders_fused(M, p):
    """1 < p < M (test_kernels.py:143-150 sweeps p = 1..4 at M = 4) on the fused kernel."""
    X = gen_brownian(6, 50, 4, SeedStream(71)).data
    Y = gen_brownian(5, 37, 4, SeedStream(72)).data
    for kind, norm, tol in (("rbf", "none", TOL_RAW), ("rbf", "levelwise", TOL_NORM),
                            ("linear", "none", TOL_RAW)):
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=M, order=p,
                           normalization=norm)
        assert uses_fast_path(50, 37, 4, cfg)
        R = O.gram(X, Y, sp=O.static_params(kind), M=M, p=p, normalization=norm)
        assert _scaled_err(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, (kind, norm)
    if M >= 6:  # multi-panel (L > 128 columns at 4 per lane) and symmetric
        X = gen_brownian(4, 300, 3, SeedStream(73)).data
        cfg = KernelConfig(n_levels=M, order=p, normalization="levelwise")
        assert uses_fast_path(300, 300, 3, cfg)
        K = sig_kernel_gram(X, cfg=cfg)
        assert np.array_equal(K, K.T) and np.array_equal(np.diag(K), np.ones(4))
        R = O.gram(X, None, sp=O.static_params("rbf"), M=M, p=p, normalization="levelwise")
        assert _scaled_err(K, R) <= TOL_NORM


@pytest.mark.parametrize("norm", ["none", "levelwise", "global"])
@pytest.mark.parametrize("kind,p", [("rbf", 1), ("linear", 1), ("rbf", 3), ("matern32", 1)])
def test_facade_diag(norm, kind, p):
    """K(X, diag=True) (north-star facade) equals the diagonal of the reference's
    K(X): unnormalised the summed self levels (kernels.py:589-590), levelwise
    (1/(M+1)) #{m: k_m(x,x) > 0}, global 1 (kernels.py:510-527)."""
    from paper_2501_07145_b200 import SignatureKernel, StaticKernel
    X = gen_brownian(7, 33, 3, SeedStream(91)).data
    X[2] = X[2, :1]  # a constant sequence: levelwise diagonal 1/(M+1)
    st = StaticKernel()
    st.spec = StaticKernelSpec(kind=kind)
    sk = SignatureKernel(n_levels=4, order=p, normalization=norm, static_kernel=st)
    got = sk(X, diag=True)
    sp = O.static_params(kind)
    want = np.diag(O.gram(X, None, sp=sp, M=4, p=p, normalization=norm))
    tol = TOL_RAW if norm == "none" else TOL_NORM
    assert got.shape == want.shape and _rel(got, want) <= tol
    if norm == "levelwise":
        assert np.array_equal(got, np.diag(sk(X)))  # bitwise the Gram's own diagonal


def _cancellation_flags(K, lv, kind, norm):
    """The certification's cancellation rule (csrc/sk_common.cuh CERT_TAU_*), on the
    FP32 K and level values: |K| < 0.05 normalised, |K| < tau sum_m |k_m| otherwise."""
    if norm != "none":
        return K.abs() < 0.05
    tau = 0.15 if kind == "linear" else 1e-2
    return K.abs() < tau * lv.abs().sum(-1)


def test_certification_flags_nothing_at_baseline_shapes():
    """The FP32 certification (sk_gram) recomputes only entries it cannot vouch for:
    at BASELINE shapes (prefix blocks) the cancellation rule flags nothing, i.e. the
    FP32 result is the result — except c4's genuinely cancelling entries (linear
    kernel, |K| below 1e-3 of sum_m |k_m|: ~4e-4 of them), which come back
    float64-exact. SK_FLAG_NO_FIXUP returns the uncertified FP32 values."""
    from paper_2501_07145_b200 import _native
    from paper_2501_07145_b200.kernels import _self_levels_t, gram_block
    for (n, L, d, M, p, kind, norm) in ((64, 50, 3, 5, 1, "rbf", "levelwise"),
                                        (96, 128, 8, 5, 5, "rbf", "none"),
                                        (96, 256, 16, 5, 1, "rbf", "levelwise"),
                                        (64, 128, 128, 3, 1, "linear", "none"),
                                        (12, 2048, 4, 8, 1, "rbf", "levelwise")):
        X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
        Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=M, order=p,
                           normalization=norm)
        dx = dy = None
        if norm != "none":
            dx = _self_levels_t(X, cfg, "fp32")
            dy = _self_levels_t(Y, cfg, "fp32")
        K0, lv = gram_block(X, Y, cfg, diag_x=dx, diag_y=dy, want_levels=True,
                            flags=_native.SK_FLAG_NO_FIXUP)
        flagged = _cancellation_flags(K0, lv, kind, norm)
        limit = 0.1 * K0.numel() if kind == "linear" else 0
        assert int(flagged.sum()) <= limit, (n, L, d, M, kind, norm)
        if flagged.any():  # the flagged entries come back float64-exact
            Kf = sig_kernel_gram(X, Y, cfg=cfg)
            K64 = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
            assert torch.allclose(Kf[flagged], K64[flagged], rtol=1e-10, atol=0)


def test_certification_fixup_recomputes_in_float64():
    """Entries the certification flags are the float64 values after the fix-up: a
    cancelling levelwise case (seed 28 of the sweep: entry 2.5e-3)."""
    from paper_2501_07145_b200 import _native
    from paper_2501_07145_b200.kernels import gram_block
    sp = dict(kind="rbf", bandwidth=1.4884218099435196)
    X = gen_brownian(5, 58, 2, SeedStream(28, ("x",))).data
    Y = gen_brownian(4, 63, 2, SeedStream(28, ("y",))).data
    cfg = KernelConfig(static=StaticKernelSpec(**sp), n_levels=8, normalization="levelwise")
    Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    K0, lv = gram_block(Xt, Yt, cfg, flags=_native.SK_FLAG_NO_FIXUP, want_levels=True)
    flagged = _cancellation_flags(K0, lv, "rbf", "levelwise").cpu().numpy()
    assert flagged.any()
    K = sig_kernel_gram(X, Y, cfg=cfg)
    K64 = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
    R = O.gram(X, Y, sp=O.static_params(**sp), M=8, p=1, normalization="levelwise")
    assert np.allclose(K[flagged], K64[flagged], rtol=1e-12, atol=0)
    assert _rel(K, R) <= TOL_NORM


@pytest.mark.parametrize("norm", ["none", "levelwise"])
def test_certification_wide_batched_redo(norm):
    """GEMM-fed path (d = 40): flagged entries are recomputed by the batched
    wide-pair float64 redo (both self pairs too when normalised) and equal the
    float64 kernel's values."""
    from paper_2501_07145_b200 import _native
    from paper_2501_07145_b200.kernels import execution_path, gram_block
    X = gen_brownian(12, 48, 40, SeedStream(91)).data
    # y ~ -x: the linear kernel's normalised levels alternate in sign and the
    # levelwise mean cancels to ~0 (flagged); plus unrelated sequences
    noise = 0.01 * gen_brownian(6, 48, 40, SeedStream(93)).data
    Y = np.concatenate([-X[:6] + noise, gen_brownian(5, 48, 40, SeedStream(92)).data])
    cfg = KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=3, normalization=norm)
    assert execution_path(48, 48, 40, cfg) == "gemm"
    Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    K0, lv = gram_block(Xt, Yt, cfg, flags=_native.SK_FLAG_NO_FIXUP, want_levels=True)
    flagged = _cancellation_flags(K0, lv, "linear", norm).cpu().numpy()
    assert flagged.any()
    K = sig_kernel_gram(X, Y, cfg=cfg)
    K64 = sig_kernel_gram(X, Y, cfg=cfg, precision="fp64")
    assert np.allclose(K[flagged], K64[flagged], rtol=1e-12, atol=0)
    R = O.gram(X, Y, sp=O.static_params("linear"), M=3, p=1, normalization=norm)
    assert _scaled_err(K, R) <= (TOL_RAW if norm == "none" else TOL_NORM)


@pytest.mark.parametrize("offset", [50.0, -1e3])
@pytest.mark.parametrize("kind,d", [("rbf", 8), ("rbf", 16), ("matern32", 4), ("rbf", 40)])
def test_offset_inputs(offset, kind, d):
    """Translation-invariant kinds are centred before the FP32 rounding (ADVICE r1:
    X + 50 used to lose 1e-3): results equal the origin-centred ones within the
    north-star tolerance, fused (d <= 16) and GEMM-fed (d = 40) paths."""
    X = gen_brownian(6, 60, d, SeedStream(5)).data + offset
    Y = gen_brownian(5, 47, d, SeedStream(6)).data + offset
    sp = O.static_params(kind)
    for norm, tol in (("levelwise", TOL_NORM), ("none", TOL_RAW)):
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=4, normalization=norm)
        R = O.gram(X, Y, sp=sp, M=4, p=1, normalization=norm)
        assert _rel(sig_kernel_gram(X, Y, cfg=cfg), R) <= tol, norm
        Rs = O.gram(X, None, sp=sp, M=4, p=1, normalization=norm)
        Ks = sig_kernel_gram(X, cfg=cfg)
        assert _rel(Ks, Rs) <= tol and np.array_equal(Ks, Ks.T), norm
