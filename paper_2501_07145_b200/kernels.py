"""Truncated signature kernels on B200: the reference-compatible boundary.

Drop-in for the reference's dual DP path (`sigkern.kernels`,
/root/reference/pkg/src/sigkern/kernels.py):

* `sig_kernel_gram` (kernels.py:530-600) — Gram matrix, symmetric or cross,
  with none/levelwise/global normalisation;
* `sig_kernel_dp` (kernels.py:307-312) — per-pair level values;
* `sig_levels_dp` (kernels.py:144-201) — level recursion on given increments;
* `increment_tensor` (kernels.py:263-281) — double-differenced point Grams.

Validation, error types and messages follow the reference. All arithmetic
runs in the CUDA library (`_native`); PyTorch only moves tensors. Inputs may
be numpy arrays / SequenceBatch (results come back as numpy, like the
reference) or torch tensors (results stay on their device).

`precision="fp32"` (default) selects the fused sm_100a FP32 kernels where a
configuration is compiled for them (rbf/linear static kernel, order 1,
n_levels <= 8, d <= 16, L <= 256 columns) and the float64 kernel otherwise;
`precision="fp64"` always uses the float64 kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from .config import KernelConfig, LevelValues, StaticKernelSpec
from .errors import ConfigError, NumericError
from .sequences import SequenceBatch
from .utils import ResourceCounters, dp_flops, gram_counts

__all__ = ["sig_kernel_gram", "sig_kernel_dp", "sig_levels_dp", "increment_tensor",
           "self_levels", "uses_fast_path", "execution_path", "sig_pde_kernel"]

ALGORITHMS = ("dp", "pde", "bruteforce")  # kernels.py:53


# ---------------------------------------------------------------------------
# tensor plumbing
# ---------------------------------------------------------------------------

def _device(device=None) -> torch.device:
    if device is not None:
        dev = torch.device(device)
        if dev.type != "cuda":
            raise RuntimeError("sigkern_b200 computes on CUDA devices only (no CPU fallback)")
        return dev
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device available: sigkern_b200 has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _as_tensor(X, dev):
    """-> (tensor float64 contiguous on dev, was_numpy)."""
    if isinstance(X, SequenceBatch):
        X = X.data
    if isinstance(X, torch.Tensor):
        return X.to(device=dev, dtype=torch.float64).contiguous(), False
    arr = np.asarray(X, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(dev), True


def _check_finite(t: torch.Tensor, what: str) -> None:
    # kernels.py:284-286
    if t.numel() and not bool(torch.isfinite(t).all()):
        raise ValueError(f"{what} contains non-finite values")


def _batch_points(X, dev):
    # kernels.py:414-422
    t, was_np = _as_tensor(X, dev)
    if t.ndim != 3:
        raise ValueError(f"expected a SequenceBatch or (N, L, d) array, got shape {tuple(t.shape)}")
    _check_finite(t, "sequence batch")
    return t, was_np


def ctypes_ptr(t):
    return None if t is None else t.data_ptr()


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _workspace(nbytes: int, dev):
    if nbytes <= 0:
        return None, 0
    return torch.empty(int(nbytes), dtype=torch.uint8, device=dev), int(nbytes)


_PATHS = {0: "fp64", 1: "fused", 2: "gemm"}


def execution_path(lx: int, ly: int, d: int, cfg: KernelConfig, precision: str = "fp32") -> str:
    """Which sm_100a path runs this configuration: "fused" (the fused FP32 Gram
    kernel, d <= 16), "gemm" (library GEMM of the cell values + the FP32
    systolic DP kernel, large d) or "fp64" (the general float64 kernel)."""
    c = _native.config_struct(cfg, precision)
    return _PATHS[_native.load().sk_fast_path(lx, ly, d, c)]


def uses_fast_path(lx: int, ly: int, d: int, cfg: KernelConfig, precision: str = "fp32") -> bool:
    """True if this configuration runs on an FP32 sm_100a path (fused or GEMM-fed)."""
    return execution_path(lx, ly, d, cfg, precision) != "fp64"


# ---------------------------------------------------------------------------
# device-level building blocks (tensors in, tensors out)
# ---------------------------------------------------------------------------

def self_levels(X, cfg: KernelConfig, precision: str = "fp32", device=None) -> torch.Tensor:
    """(N, M+1) self level values k_m(x_i, x_i) (kernels.py:589-595)."""
    dev = _device(device) if not isinstance(X, torch.Tensor) or not X.is_cuda else X.device
    Xt, _ = _batch_points(X, dev)
    return _self_levels_t(Xt, cfg, precision)


def _self_levels_t(Xt: torch.Tensor, cfg: KernelConfig, precision: str,
                   c=None, ws=None, flags: int = 0) -> torch.Tensor:
    lib = _native.load()
    dev = Xt.device
    n, L, d = Xt.shape
    M = cfg.n_levels
    out = torch.empty((n, M + 1), dtype=torch.float64, device=dev)
    if n == 0:
        return out
    c = c or _native.config_struct(cfg, precision, flags)
    with torch.cuda.device(dev):  # workspace sizes depend on the device's SM count
        if ws is None:
            ws = _workspace(lib.sk_workspace_bytes(n, L, 0, 0, d, c), dev)
        buf, nb = ws
        rc = lib.sk_self_levels(Xt.data_ptr(), n, L, d, c, out.data_ptr(),
                                ctypes_ptr(buf), nb, _stream(dev))
    _native.check(rc, "sk_self_levels")
    return out


def gram_block(Xt: torch.Tensor, Yt: torch.Tensor | None, cfg: KernelConfig,
               row_begin: int = 0, row_end: int | None = None, precision: str = "fp32",
               diag_x=None, diag_y=None, K=None, want_levels: bool = False,
               check_global: bool = True, flags: int = 0):
    """Rows [row_begin, row_end) of the Gram on device tensors (the sk_gram call).

    Yt=None is the symmetric K(X): K must then be the full (N, N) matrix (it is
    allocated if omitted) and only pairs i <= j with i in the row range are
    evaluated and mirrored. Returns (K, levels-or-None). `flags`:
    `_native.SK_FLAG_NO_FIXUP` leaves the FP32 certification's NaN markers in
    K (diagnostics; see include/sigkern_b200.h).
    """
    lib = _native.load()
    dev = Xt.device
    sym = Yt is None
    nx, lx, d = Xt.shape
    ny, ly = (nx, lx) if sym else Yt.shape[:2]
    row_end = nx if row_end is None else row_end
    M = cfg.n_levels
    c = _native.config_struct(cfg, precision, flags)
    with torch.cuda.device(dev):  # workspace sizes depend on the device's SM count
        ws = _workspace(lib.sk_workspace_bytes(nx, lx, ny, ly, d, c), dev)
    if cfg.normalization != "none":
        if diag_x is None:
            diag_x = _self_levels_t(Xt, cfg, precision, c, ws)
        if diag_y is None:
            diag_y = diag_x if sym else _self_levels_t(Yt, cfg, precision, c, ws)
        if cfg.normalization == "global" and check_global:
            _check_global(diag_x, diag_y)
    rows = nx if sym else row_end - row_begin
    if K is None:
        K = torch.empty((rows, ny), dtype=torch.float64, device=dev)
    lv = torch.empty((rows, ny, M + 1), dtype=torch.float64, device=dev) if want_levels else None
    if nx and ny and row_end > row_begin:
        with torch.cuda.device(dev):
            rc = lib.sk_gram(Xt.data_ptr(), nx, lx, ctypes_ptr(Xt if sym else Yt), ny, ly, d,
                             1 if sym else 0, c, row_begin, row_end, ctypes_ptr(diag_x),
                             ctypes_ptr(diag_y), K.data_ptr(), K.stride(0),
                             ctypes_ptr(lv), ctypes_ptr(ws[0]), ws[1], _stream(dev))
        _native.check(rc, "sk_gram")
    return K, lv


def _check_global(diag_x, diag_y) -> None:
    # kernels.py:519-527 (checked before the Gram; same exception and message)
    sx = diag_x.sum(dim=-1)
    sy = diag_y.sum(dim=-1)
    bad_x = torch.nonzero(sx <= 0).flatten()
    bad_y = torch.nonzero(sy <= 0).flatten()
    if bad_x.numel() or bad_y.numel():
        which = bad_x if bad_x.numel() else bad_y
        raise NumericError(
            f"global normalization undefined: non-positive self-kernel for "
            f"input sequence index {int(which[0])}")


# ---------------------------------------------------------------------------
# reference-compatible public functions
# ---------------------------------------------------------------------------

def sig_kernel_gram(X, Y=None, cfg: KernelConfig = None, algorithm: str = "dp",
                    n_threads: int = 1, counters=None, tile_memory: int = 256 * 2 ** 20,
                    *, precision: str = "fp32", device=None):
    """Pairwise signature-kernel matrix (kernels.py:530-600).

    X, Y: SequenceBatch / (N, L, d) arrays or tensors; Y=None is K(X, X),
    evaluated on the upper triangle and mirrored bit for bit. `n_threads`
    and `tile_memory` are accepted for compatibility; as in the reference,
    results do not depend on them.
    """
    if cfg is None:
        cfg = KernelConfig()
    if algorithm not in ALGORITHMS:
        raise ValueError(f"algorithm must be one of {ALGORITHMS}, got {algorithm!r}")
    if algorithm == "pde" and cfg.normalization == "levelwise":
        raise ConfigError(
            "kernel.normalization: levelwise normalization requires level values; "
            "the pde algorithm supports none/global")
    if algorithm == "bruteforce":
        raise NotImplementedError(
            "algorithm='bruteforce' is the reference's test oracle (kernels.py:218-249) and is "
            "not part of the B200 build")
    if counters is None:
        counters = ResourceCounters()
    dev = X.device if isinstance(X, torch.Tensor) and X.is_cuda else _device(device)
    Xt, was_np = _batch_points(X, dev)
    sym = Y is None
    Yt = None if sym else _batch_points(Y, dev)[0]
    dy = Xt.shape[2] if sym else Yt.shape[2]
    if Xt.shape[2] != dy:
        raise ValueError(f"channel mismatch: d={Xt.shape[2]} vs d={dy}")
    if algorithm == "pde":
        K = pde_gram_block(Xt, Yt, cfg)
        _count(counters, Xt, Yt, cfg, K, "pde", tile_memory)
        return K.cpu().numpy() if was_np else K
    K, _ = gram_block(Xt, Yt, cfg, precision=precision)
    _count(counters, Xt, Yt, cfg, K, "dp", tile_memory)
    return K.cpu().numpy() if was_np else K


# ---------------------------------------------------------------------------
# algorithm="pde": untruncated signature kernel (kernels.py:334-507), float64
# ---------------------------------------------------------------------------

def _pde_self_t(Xt: torch.Tensor, cfg: KernelConfig) -> torch.Tensor:
    lib = _native.load()
    n, L, d = Xt.shape
    out = torch.empty(n, dtype=torch.float64, device=Xt.device)
    if n == 0:
        return out
    buf, nb = _workspace(lib.sk_pde_workspace_bytes(n, L, int(cfg.difference)), Xt.device)
    sp = _native.static_struct(cfg.static)
    with torch.cuda.device(Xt.device):
        rc = lib.sk_pde_self(Xt.data_ptr(), n, L, d, sp, int(cfg.difference), out.data_ptr(),
                             ctypes_ptr(buf), nb, _stream(Xt.device))
    _native.check(rc, "sk_pde_self")
    return out


def pde_gram_block(Xt: torch.Tensor, Yt: torch.Tensor | None, cfg: KernelConfig) -> torch.Tensor:
    """Goursat-PDE Gram on device tensors (the reference's _pde_gram + global
    normalisation, kernels.py:559-571)."""
    lib = _native.load()
    sym = Yt is None
    nx, lx, d = Xt.shape
    Ys = Xt if sym else Yt
    ny, ly = Ys.shape[0], Ys.shape[1]
    if cfg.difference and (lx < 2 or ly < 2) and nx and ny:
        raise ValueError("pde kernel needs at least one increment per sequence")
    K = torch.zeros((nx, ny), dtype=torch.float64, device=Xt.device)
    if nx and ny:
        buf, nb = _workspace(lib.sk_pde_workspace_bytes(nx * ny, ly, int(cfg.difference)),
                             Xt.device)
        sp = _native.static_struct(cfg.static)
        with torch.cuda.device(Xt.device):
            rc = lib.sk_pde_gram(Xt.data_ptr(), nx, lx, Ys.data_ptr(), ny, ly, d, int(sym), sp,
                                 int(cfg.difference), 0, nx, K.data_ptr(), ny, ctypes_ptr(buf),
                                 nb, _stream(Xt.device))
        _native.check(rc, "sk_pde_gram")
    if cfg.normalization == "global":
        sx = _pde_self_t(Xt, cfg)
        sy = sx if sym else _pde_self_t(Yt, cfg)
        for s in (sx, sy):  # kernels.py:519-527
            bad = torch.nonzero(s <= 0).flatten()
            if bad.numel():
                raise NumericError(
                    f"global normalization undefined: non-positive self-kernel for "
                    f"input sequence index {int(bad[0])}")
        K = K / torch.sqrt(sx[:, None] * sy[None, :])
    return K


def sig_pde_kernel(x, y, cfg: KernelConfig, counters=None, *, device=None) -> float:
    """Untruncated signature kernel of one pair via the PDE solve (kernels.py:405-411)."""
    dev = _device(device)
    xt, _ = _as_pair_points(x, dev)
    yt, _ = _as_pair_points(y, dev)
    if xt.shape[1] != yt.shape[1]:
        raise ValueError(f"dimension mismatch: {xt.shape[1]} vs {yt.shape[1]}")
    K = pde_gram_block(xt[None], yt[None], KernelConfig(
        static=cfg.static, n_levels=cfg.n_levels, order=cfg.order, difference=cfg.difference,
        normalization="none"))
    return float(K[0, 0])


def _count(counters, Xt, Yt, cfg, K, algorithm, tile_memory):
    """The reference's analytic counts for this call (utils.gram_counts) and the
    device's own footprint (inputs, packed FP32 roles, K)."""
    nx, lx, d = Xt.shape
    ny, ly = (nx, lx) if Yt is None else Yt.shape[:2]
    gram_counts(counters, nx, lx, ny, ly, d, cfg.n_levels, cfg.effective_order,
                bool(cfg.difference), cfg.normalization, Yt is None, algorithm, tile_memory)
    if hasattr(counters, "observe_device_bytes"):
        counters.observe_device_bytes(
            K.numel() * 8 + (Xt.numel() + (0 if Yt is None else Yt.numel())) * 12)


def _as_pair_points(x, dev):
    # kernels.py:289-296
    t, was_np = _as_tensor(x, dev)
    if t.ndim == 1:
        t = t[:, None]
    if t.ndim != 2:
        raise ValueError(f"a sequence must be a (L, d) array, got shape {tuple(t.shape)}")
    _check_finite(t, "sequence")
    return t, was_np


def sig_kernel_dp(x, y, cfg: KernelConfig, counters=None, *, precision: str = "fp64",
                  device=None) -> LevelValues:
    """Level kernels k_0..k_M of one pair (kernels.py:307-312).

    Float64 by default, like the reference's per-pair values: a single pair
    gains nothing from the FP32 Gram kernels."""
    dev = _device(device)
    xt, _ = _as_pair_points(x, dev)
    yt, _ = _as_pair_points(y, dev)
    if xt.shape[1] != yt.shape[1]:
        raise ValueError(f"dimension mismatch: {xt.shape[1]} vs {yt.shape[1]}")
    _, lv = gram_block(xt[None], yt[None], KernelConfig(
        static=cfg.static, n_levels=cfg.n_levels, order=cfg.order,
        difference=cfg.difference, normalization="none"), precision=precision, want_levels=True)
    if counters is not None:
        T1 = xt.shape[0] - 1 if cfg.difference else xt.shape[0]
        T2 = yt.shape[0] - 1 if cfg.difference else yt.shape[0]
        counters.add_flops(dp_flops(1, max(T1, 0), max(T2, 0), xt.shape[1], cfg.n_levels,
                                    cfg.effective_order, cfg.difference))
    return LevelValues(lv[0, 0].cpu().numpy())


def sig_levels_dp(mats, n_levels: int, order: int = 1, counters=None, *, device=None):
    """Level values from increment matrices (kernels.py:144-201), float64 on device.

    mats: one (..., T1, T2) array shared by all levels or a list of n_levels
    arrays (level m uses mats[m-1], kernels.py:129-141). Returns
    (..., n_levels+1) with [..., 0] = 1, numpy in / numpy out.
    """
    M = int(n_levels)
    dev = _device(device)
    per_level = isinstance(mats, (list, tuple))
    if per_level and M >= 1:
        if len(mats) != M:
            raise ValueError(
                f"per-level increment list must have n_levels={M} entries, got {len(mats)}")
        arrs = [_as_tensor(m, dev)[0] for m in mats]
        shapes = {tuple(a.shape) for a in arrs}
        if len(shapes) > 1:
            raise ValueError(f"per-level increment matrices disagree on shape: {shapes}")
        was_np = not isinstance(mats[0], torch.Tensor)
        A = torch.stack(arrs)  # (M, ..., T1, T2)
        first_shape = arrs[0].shape
    else:
        raw = mats[0] if per_level and len(mats) else mats
        A, was_np = _as_tensor(raw, dev)
        if A.ndim < 2:
            A = A.reshape(0, 0)
        per_level = False
        first_shape = A.shape
    lead = tuple(first_shape[:-2])
    T1, T2 = int(first_shape[-2]), int(first_shape[-1])
    batch = int(np.prod(lead, dtype=np.int64)) if lead else 1
    out = torch.zeros((batch, M + 1), dtype=torch.float64, device=dev)
    out[:, 0] = 1.0
    p = max(1, min(int(order), M)) if M >= 1 else 1
    if M >= 1 and T1 > 0 and T2 > 0 and batch > 0:
        lib = _native.load()
        A = A.reshape((M, batch, T1, T2) if per_level else (batch, T1, T2)).contiguous()
        buf, nb = _workspace(lib.sk_levels_dp_workspace_bytes(batch, T1, T2, M, p), dev)
        with torch.cuda.device(dev):
            rc = lib.sk_levels_dp(A.data_ptr(), batch, T1, T2, M, p, 1 if per_level else 0,
                                  out.data_ptr(), ctypes_ptr(buf), nb, _stream(dev))
        _native.check(rc, "sk_levels_dp")
    if counters is not None:
        counters.add_flops(dp_flops(batch, T1, T2, 0, M, p, False))
    out = out.reshape(lead + (M + 1,))
    return out.cpu().numpy() if was_np else out


def increment_tensor(spec: StaticKernelSpec, X, Y, difference: bool = True, counters=None,
                     *, device=None):
    """Increment matrices of (batched) point arrays (..., L, d) (kernels.py:263-281).

    Leading axes broadcast as in the reference. Float64 on device.
    """
    dev = _device(device)
    Xt, was_np = _as_tensor(X, dev)
    Yt, _ = _as_tensor(Y, dev)
    if Xt.ndim < 2 or Yt.ndim < 2:
        raise ValueError("increment_tensor expects (..., L, d) point arrays")
    if Xt.shape[-1] != Yt.shape[-1]:
        raise ValueError(f"dimension mismatch: d={Xt.shape[-1]} vs d={Yt.shape[-1]}")
    lead = torch.broadcast_shapes(Xt.shape[:-2], Yt.shape[:-2])
    L1, L2, d = Xt.shape[-2], Yt.shape[-2], Xt.shape[-1]
    Xe = Xt.expand(lead + (L1, d)).reshape(-1, L1, d).contiguous()
    Ye = Yt.expand(lead + (L2, d)).reshape(-1, L2, d).contiguous()
    n = Xe.shape[0]
    T1 = max(L1 - 1, 0) if difference else L1
    T2 = max(L2 - 1, 0) if difference else L2
    out = torch.zeros((n, T1, T2), dtype=torch.float64, device=dev)
    if n and T1 and T2:
        lib = _native.load()
        sp = _native.static_struct(spec)
        with torch.cuda.device(dev):
            rc = lib.sk_increment_tensor(Xe.data_ptr(), n, L1, Ye.data_ptr(), n, L2, d, 1, sp,
                                         1 if difference else 0, out.data_ptr(), _stream(dev))
        _native.check(rc, "sk_increment_tensor")
    if counters is not None:
        counters.add_flops(n * L1 * L2 * d + (3 * T1 * T2 * n if difference else 0))
    out = out.reshape(tuple(lead) + (T1, T2))
    return out.cpu().numpy() if was_np else out

