"""C-ABI library: loads without a GPU, exports every symbol the header declares,
and its host-side logic (validation, fast-path selection, workspace sizing)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_2501_07145_b200 import KernelConfig, StaticKernelSpec, _native

HEADER = os.path.join(ROOT, "include", "sigkern_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SK_API\s+(?:const\s+char\s*\*|int|size_t)\s*(sk_\w+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    lib = _native.load()
    names = _declared()
    assert names, "no SK_API declarations parsed"
    assert set(names) == set(_native.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n
    c5 = _native.config_struct(KernelConfig(n_levels=8))
    # few sequences: the certification scratch is the larger part
    assert lib.sk_workspace_bytes(2, 256, 2, 256, 4, c5) == 256 + cert_bytes(2, 256, 2, 256, 4, 8)
    assert lib.sk_abi_version() == 2
    assert lib.sk_last_error() == b""


def _cfg(**kw):
    st = kw.pop("static", StaticKernelSpec(kind="rbf"))
    prec = kw.pop("precision", "fp32")
    return _native.config_struct(KernelConfig(static=st, **kw), prec)


def test_fast_path_selection():
    lib = _native.load()
    c3 = _native.config_struct(KernelConfig(n_levels=5, order=1, normalization="levelwise"))
    assert lib.sk_fast_path(256, 256, 16, c3) == 1          # c3
    assert lib.sk_fast_path(50, 50, 3, c3) == 1             # c1 shapes
    lin = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=3))
    assert lib.sk_fast_path(128, 128, 16, lin) == 1
    assert lib.sk_fast_path(128, 128, 128, lin) == 2        # d > 16: GEMM-fed path (c4)
    geo24 = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=5,
                                               order=3))
    assert lib.sk_fast_path(64, 64, 24, geo24) == 2         # GEMM-fed, 1 < p < M
    assert lib.sk_fast_path(64, 64, 24, _native.config_struct(KernelConfig())) == 0  # rbf d > 16
    assert lib.sk_fast_path(1000, 1000, 16, lin) == 2       # x ring too large for shared memory
    geo = _native.config_struct(KernelConfig(n_levels=5, order=5))
    assert lib.sk_fast_path(128, 128, 8, geo) == 1          # geometric p = M (c2)
    mid = _native.config_struct(KernelConfig(n_levels=5, order=3))
    assert lib.sk_fast_path(128, 128, 8, mid) == 1          # 1 < p < M: fused general order
    for M, p in ((6, 2), (6, 3), (7, 2), (8, 2)):             # many levels, low order: fused
        assert lib.sk_fast_path(128, 128, 8, _native.config_struct(KernelConfig(n_levels=M, order=p))) == 1
    big = _native.config_struct(KernelConfig(n_levels=6, order=4))
    assert lib.sk_fast_path(128, 128, 8, big) == 0          # register budget exceeded: float64
    lgeo = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=4,
                                              order=4, normalization="levelwise"))
    assert lib.sk_fast_path(64, 64, 4, lgeo) == 0           # normalised linear p > 1: float64
    f64 = _native.config_struct(KernelConfig(n_levels=5), "fp64")
    assert lib.sk_fast_path(256, 256, 16, f64) == 0
    mat = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="matern32")))
    assert lib.sk_fast_path(64, 64, 4, mat) == 1            # stationary kinds, order 1: fused
    matp = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="matern32"), n_levels=3,
                                              order=3))
    assert lib.sk_fast_path(64, 64, 4, matp) == 1           # stationary kinds, order > 1: fused
    poly = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="polynomial")))
    assert lib.sk_fast_path(64, 64, 4, poly) == 0           # polynomial: float64
    poly2 = _native.config_struct(KernelConfig(static=StaticKernelSpec(kind="polynomial"),
                                               n_levels=3, order=2))
    assert lib.sk_fast_path(64, 64, 4, poly2) == 0          # polynomial, order > 1: float64
    assert lib.sk_fast_path(300, 300, 4, c3) == 1           # two 256-column panels
    assert lib.sk_fast_path(2048, 2048, 4, _native.config_struct(KernelConfig(n_levels=8))) == 1  # c5
    assert lib.sk_fast_path(1000, 1000, 16, c3) == 0        # rbf, x ring beyond shared memory: float64
    assert lib.sk_fast_path(2, 256, 4, c3) == 0             # x shorter than the wavefront


def _a256(b):
    return (b + 255) // 256 * 256


def cert_bytes(nx, lx, ny, ly, d, M):
    # corner points of both roles (scan) or per-CTA float64 slots (redo: 4 CTAs
    # per SM, row buffer + (M-1) column accumulators), then the compacted list
    # of flagged entries (a count + up to min(nx*ny, 4 Mi) indices)
    L = max(lx, ly)
    slot = L + 2 + (M - 1) * (L - 1)
    redo = min(148 * 4, (256 << 20) // (slot * 8)) * slot * 8
    corners = (nx + ny) * 2 * d * 8
    return _a256(max(redo, corners)) + _a256((min(nx * ny, 1 << 22) + 1) * 8)


def test_workspace_sizes():
    lib = _native.load()
    c3 = _native.config_struct(KernelConfig(n_levels=5, normalization="levelwise"))
    n, L, d = 8192, 256, 16
    ws = lib.sk_workspace_bytes(n, L, n, L, d, c3)
    # the certification's per-entry (FP32 level 1, sum |k_m|) float pair, then the
    # larger of the packed roles (x row pairs of 2*16+4 floats, y points of 16+4
    # floats, the midrange codes of the centring: 2d u64, 256-byte aligned) and
    # the certification scratch (sk_rowscan.cu cert_workspace_bytes)
    roles = n * (L // 2) * 36 * 4 + n * L * 20 * 4 + 256
    assert ws == n * n * 8 + max(roles, cert_bytes(n, L, n, L, d, 5))
    assert lib.sk_abi_version() == 2
    f64 = _native.config_struct(KernelConfig(n_levels=3, order=2), "fp64")
    assert lib.sk_workspace_bytes(4, 6, 5, 7, 2, f64) > 0


def test_invalid_arguments_rejected_before_device_work():
    lib = _native.load()
    bad = _native.config_struct(KernelConfig(n_levels=3))
    bad.order = 9  # effective order must be <= n_levels
    rc = lib.sk_gram(None, 0, 5, None, 0, 5, 2, 0, ctypes.byref(bad), 0, 0, None, None,
                     None, 0, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID
    assert b"order" in lib.sk_last_error()
    good = _native.config_struct(KernelConfig(n_levels=3, normalization="levelwise"))
    rc = lib.sk_gram(None, 0, 5, None, 0, 5, 2, 0, ctypes.byref(good), 0, 0, None, None,
                     None, 0, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID  # neither K nor levels
    rc = lib.sk_levels_dp(None, 1, 2, 2, 17, 1, 0, None, None, 0, None)
    assert rc == _native.SK_ERR_UNSUPPORTED
    with pytest.raises(ValueError):
        _native.check(_native.SK_ERR_INVALID, "x")


def test_rfsf_entry_points_validate_on_the_host():
    """sk_static_features / sk_lifted_gram / sk_lifted_self_levels reject bad
    arguments before any device work (features.py:446-475 boundary)."""
    lib = _native.load()
    fm = _native.SkFeatureMap(7, 0, 4, 8, None, None, None, None, _native.SkStaticSpec(2, 3, 1.0, 1.0, 1.0, 1.0))
    assert lib.sk_static_features(fm, None, 3, 2, None, 8, None, 0, None) == _native.SK_ERR_INVALID
    assert b"unknown feature kind" in lib.sk_last_error()
    fm.kind = 0  # rff: out_dim must be 2 D
    fm.out_dim = 5
    assert lib.sk_static_features(fm, None, 3, 2, None, 8, None, 0, None) == _native.SK_ERR_INVALID
    assert b"out_dim" in lib.sk_last_error()
    fm.out_dim = 8
    assert lib.sk_static_features(fm, None, 3, 2, None, 8, None, 0, None) == _native.SK_ERR_INVALID
    assert b"NULL" in lib.sk_last_error() or b"weights" in lib.sk_last_error()
    assert lib.sk_static_features(fm, None, 0, 2, None, 8, None, 0, None) == _native.SK_OK  # empty
    assert lib.sk_static_features_workspace_bytes(fm, 100) == 0
    fm.kind, fm.out_dim = 2, 3  # nystroem: n x D landmark Gram in the workspace
    assert lib.sk_static_features_workspace_bytes(fm, 100) == 100 * 4 * 8
    offs = (ctypes.c_int64 * 4)(0, 2, 4, 6)
    args = dict(nx=2, lx=5, ny=2, ly=5, width=6)
    rc = lib.sk_lifted_gram(None, 2, 5, None, 2, 5, 6, offs, 3, 4, 1, 0, 0, 0, 2, None, None,
                            None, 2, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID and b"order" in lib.sk_last_error()
    rc = lib.sk_lifted_gram(None, 2, 5, None, 2, 5, 6, None, 3, 1, 1, 0, 0, 0, 2, None, None,
                            None, 2, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID and b"slot_offsets" in lib.sk_last_error()
    rc = lib.sk_lifted_gram(None, 2, 5, None, 2, 5, 6, offs, 3, 1, 1, 1, 0, 0, 2, None, None,
                            None, 2, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID  # UX is NULL
    rc = lib.sk_lifted_self_levels(None, 2, 5, 6, offs, -1, 1, 1, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID and b"n_levels" in lib.sk_last_error()
    full = lib.sk_lifted_gram_workspace_bytes(args["nx"], args["lx"], args["ny"], args["ly"], 3, 1, 1)
    small = lib.sk_lifted_workspace_bytes(4, 5, 3, 1, 1)
    assert full > small > 0
    assert lib.sk_lifted_gram_workspace_bytes(0, 5, 2, 5, 3, 1, 1) == 0


def test_pde_and_pairwise_entry_points_validate_on_the_host():
    lib = _native.load()
    sp = _native.SkStaticSpec(99, 3, 1.0, 1.0, 1.0, 1.0)
    rc = lib.sk_pde_gram(None, 1, 4, None, 1, 4, 2, 0, ctypes.byref(sp), 1, 0, 1, None, 1, None, 0, None)
    assert rc == _native.SK_ERR_INVALID and b"kind" in lib.sk_last_error()
    sp.kind = 2
    rc = lib.sk_pde_self(None, 1, 1, 2, ctypes.byref(sp), 1, None, None, 0, None)
    assert rc == _native.SK_ERR_INVALID  # X NULL / one point with difference=True
    assert lib.sk_pairwise_dist(None, 4, 0, None, None) == _native.SK_ERR_INVALID
    assert lib.sk_pairwise_dist(None, 1, 3, None, None) == _native.SK_OK  # no pairs
    assert lib.sk_pde_workspace_bytes(10, 5, 1) > 0
