"""Exact Gram of a fitted `rfsf_full` random-feature map (features.py:397-475).

`rfsf_exact_gram(state, X, Y=None, normalize=False)` evaluates
<Phi(x), Phi(y)> of the rfsf_full signature feature map without ever forming
the (2D)^m-wide features: level m of the dual DP runs with the static kernel
replaced by the inner product of slot m's static features (the finite-rank
lift, `_lifted_level_grams`, features.py:397-424). On the device this is

  1. `sk_static_features` per slot (transform_static_features,
     static/features.py:102-124: rff, rff1d, nystroem), written side by side
     into one (N, L, sum_a w_a) float64 buffer, and
  2. `sk_lifted_gram`: the float64 level recursion with a per-level point
     kernel (each cell double-differences M slot inner products).

`state` may be the reference's own `SigFeatureState` (duck-typed: `config`
with variant/n_levels/effective_order/difference, and `slot_states` with
spec/weights/phases/landmarks/whiten) or the mirror types below, whose
`fit_sig_features` reproduces the reference's sampling for the static slots
bit for bit (same SeedStream children `level{a}`, features.py:167-194).
The primal feature maps themselves (transform_sig_features, the trp/ts
projections) are not part of this path.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native
from .config import StaticKernelSpec
from .kernels import _as_tensor, _device, _stream, _workspace, ctypes_ptr, increment_tensor
from .sequences import SeedStream, SequenceBatch
from .utils import ResourceCounters, dp_flops

__all__ = ["StaticFeatureSpec", "StaticFeatureState", "SigFeatureConfig", "SigFeatureState",
           "fit_static_features", "fit_sig_features", "transform_static_features",
           "rfsf_exact_gram", "FEATURE_KINDS", "VARIANTS"]

FEATURE_KINDS = ("rff", "rff1d", "nystroem")  # static/features.py:32
VARIANTS = ("rfsf_full", "dp", "dp1d", "trp", "ts")  # features.py:58
EIGENVALUE_FLOOR = 1e-12  # static/features.py:35
_FEAT_CODES = {"rff": 0, "rff1d": 1, "nystroem": 2}


@dataclass(frozen=True)
class StaticFeatureSpec:
    """static/features.py:40-53."""

    kind: str = "rff"
    n_components: int = 100
    bandwidth: float = 1.0
    base_kernel: StaticKernelSpec = field(default_factory=StaticKernelSpec)

    def __post_init__(self):
        if self.kind not in FEATURE_KINDS:
            raise ValueError(f"unknown feature kind {self.kind!r}; choose from {FEATURE_KINDS}")
        if not (isinstance(self.n_components, (int, np.integer)) and self.n_components >= 1):
            raise ValueError(f"n_components must be a positive integer, got {self.n_components}")
        if not self.bandwidth > 0:
            raise ValueError(f"bandwidth must be positive, got {self.bandwidth}")


@dataclass
class StaticFeatureState:
    """static/features.py:56-66."""

    spec: StaticFeatureSpec
    input_dim: int
    out_dim: int
    weights: np.ndarray = None  # (d, D)
    phases: np.ndarray = None  # (D,)
    landmarks: np.ndarray = None  # (D, d)
    whiten: np.ndarray = None  # (D, out_dim)


@dataclass(frozen=True)
class SigFeatureConfig:
    """features.py:62-112 (the fields rfsf_exact_gram reads, same validation)."""

    variant: str = "trp"
    static: StaticFeatureSpec = field(default_factory=StaticFeatureSpec)
    n_components: int = 100
    projection: int = 100
    n_levels: int = 5
    order: int | None = 1
    difference: bool = True
    normalize: bool = False

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}; choose from {VARIANTS}")
        for name in ("n_components", "projection"):
            v = getattr(self, name)
            if not (isinstance(v, (int, np.integer)) and v >= 1):
                raise ValueError(f"{name} must be a positive integer, got {v}")
        if not (isinstance(self.n_levels, (int, np.integer)) and self.n_levels >= 0):
            raise ValueError(f"n_levels must be a non-negative integer, got {self.n_levels}")
        if self.order is not None and not (
                isinstance(self.order, (int, np.integer)) and self.order >= 1):
            raise ValueError(f"order must be a positive integer or None, got {self.order}")
        allowed = {"rfsf_full": ("rff", "nystroem"), "trp": ("rff",), "ts": ("rff",),
                   "dp": ("rff",), "dp1d": ("rff1d",)}[self.variant]
        if self.static.kind not in allowed:
            raise ValueError(
                f"variant {self.variant!r} requires a static feature kind in {allowed}, "
                f"got {self.static.kind!r}")

    @property
    def effective_order(self) -> int:
        if self.n_levels == 0:
            return 1
        if self.order is None:
            return self.n_levels
        return min(int(self.order), self.n_levels)


@dataclass
class SigFeatureState:
    """features.py:114-123."""

    config: SigFeatureConfig
    input_dim: int
    slot_states: list
    proj_states: list | None
    level_dims: list


def fit_static_features(spec: StaticFeatureSpec, train, seed: SeedStream,
                        device=None) -> StaticFeatureState:
    """Sample a static feature map (static/features.py:69-99). Host-side setup;
    the nystroem landmark Gram is evaluated on the device."""
    train = np.atleast_2d(np.asarray(train, dtype=np.float64))
    d = train.shape[1]
    D = spec.n_components
    rng = seed.generator()
    if spec.kind == "rff":
        W = rng.standard_normal((d, D)) / spec.bandwidth
        return StaticFeatureState(spec, d, 2 * D, weights=W)
    if spec.kind == "rff1d":
        W = rng.standard_normal((d, D)) / spec.bandwidth
        b = rng.uniform(0.0, 2.0 * math.pi, D)
        return StaticFeatureState(spec, d, D, weights=W, phases=b)
    n = train.shape[0]
    if n < D:
        raise ValueError(f"nystroem needs at least n_components={D} training vectors, got {n}")
    idx = rng.choice(n, size=D, replace=False)
    Z = train[np.sort(idx)]
    # landmark Gram k(z_i, z_j) on the device (raw point kernel, difference=False)
    K = increment_tensor(spec.base_kernel, Z[None], Z[None], difference=False,
                         device=device)[0]
    evals, evecs = np.linalg.eigh(np.asarray(K))
    keep = evals > EIGENVALUE_FLOOR
    evals = evals[keep]
    evecs = evecs[:, keep]
    return StaticFeatureState(spec, d, int(evals.shape[0]), landmarks=Z,
                              whiten=evecs / np.sqrt(evals))


def fit_sig_features(cfg: SigFeatureConfig, train, seed: SeedStream,
                     device=None) -> SigFeatureState:
    """Static slots of a signature feature map (features.py:167-194); the
    trp/ts projection slots are outside this path."""
    if cfg.variant in ("trp", "ts"):
        raise NotImplementedError(
            f"variant {cfg.variant!r} needs random projections, which are not on the "
            "exact-Gram path; only the static slots are fitted here")
    if isinstance(train, SequenceBatch):
        train = train.data
    arr = np.asarray(train, dtype=np.float64)
    pts = arr.reshape(-1, arr.shape[-1])
    spec = replace(cfg.static, n_components=cfg.n_components)
    M = cfg.n_levels
    slots = [fit_static_features(spec, pts, seed.child(f"level{a}"), device=device)
             for a in range(1, M + 1)]
    dims = [s.out_dim for s in slots]
    level_dims = [1]
    for m in range(1, M + 1):
        if cfg.variant == "rfsf_full":
            level_dims.append(int(np.prod(dims[:m], dtype=np.int64)))
        elif cfg.variant == "dp":
            level_dims.append((2 ** m) * cfg.n_components)
        else:
            level_dims.append(cfg.n_components)
    return SigFeatureState(cfg, pts.shape[1], slots, None, level_dims)


def _map_struct(st, dev):
    """-> (SkFeatureMap, keep-alive device tensors) for a fitted slot state."""
    spec = st.spec
    kind = spec.kind
    if kind not in _FEAT_CODES:
        raise ValueError(f"unknown feature kind {kind!r}; choose from {FEATURE_KINDS}")
    t = lambda a: None if a is None else torch.as_tensor(  # noqa: E731
        np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    W, b, Z, Wh = t(st.weights), t(st.phases), t(st.landmarks), t(st.whiten)
    base = _native.static_struct(spec.base_kernel) if kind == "nystroem" \
        else _native.SkStaticSpec(0, 1, 1.0, 1.0, 1.0, 1.0)
    m = _native.SkFeatureMap(_FEAT_CODES[kind], 0, int(spec.n_components), int(st.out_dim),
                             ctypes_ptr(W), ctypes_ptr(b), ctypes_ptr(Z), ctypes_ptr(Wh), base)
    return m, (W, b, Z, Wh)


def _transform_into(st, Xt: torch.Tensor, out: torch.Tensor, col: int) -> None:
    """Slot features of every point of Xt (n, L, d) into out[..., col:col+out_dim]."""
    if Xt.shape[-1] != st.input_dim:
        raise ValueError(f"dimension mismatch: fitted on d={st.input_dim}, got d={Xt.shape[-1]}")
    lib = _native.load()
    dev = Xt.device
    m, keep = _map_struct(st, dev)
    npts = Xt.numel() // Xt.shape[-1]
    buf, nb = _workspace(lib.sk_static_features_workspace_bytes(m, npts), dev)
    dst = out.view(-1, out.shape[-1])
    with torch.cuda.device(dev):
        rc = lib.sk_static_features(m, Xt.data_ptr(), npts, Xt.shape[-1],
                                    dst.data_ptr() + 8 * col, dst.shape[1], ctypes_ptr(buf),
                                    nb, _stream(dev))
    _native.check(rc, "sk_static_features")
    del keep


def transform_static_features(state, X, counters=None, *, device=None):
    """Map rows of X (..., d) to feature space (..., out_dim)
    (static/features.py:102-124), float64 on the device; numpy in, numpy out."""
    dev = _device(device)
    Xt, was_np = _as_tensor(X, dev)
    if Xt.ndim == 0 or Xt.shape[-1] != state.input_dim:
        raise ValueError(f"dimension mismatch: fitted on d={state.input_dim}, "
                         f"got d={Xt.shape[-1] if Xt.ndim else 0}")
    lead = tuple(Xt.shape[:-1])
    out = torch.empty(lead + (int(state.out_dim),), dtype=torch.float64, device=dev)
    if out.numel():
        _transform_into(state, Xt.reshape(-1, 1, Xt.shape[-1]), out.view(-1, 1, out.shape[-1]), 0)
    if counters is not None:
        counters.add_flops(_transform_flops(state, int(np.prod(lead, dtype=np.int64))))
    return out.cpu().numpy() if was_np else out


def _transform_flops(st, npts: int) -> int:
    spec = st.spec
    D = spec.n_components
    if spec.kind == "rff":
        return npts * D * st.input_dim + 2 * npts * D
    if spec.kind == "rff1d":
        return npts * D * st.input_dim + npts * D
    return npts * D * (st.input_dim + st.out_dim)


def _lift(state, Xt: torch.Tensor):
    """-> (U (n, L, W) float64, slot offsets (M+1,) int64) of every slot's features."""
    slots = state.slot_states
    widths = [int(s.out_dim) for s in slots]
    offs = np.concatenate([[0], np.cumsum(widths)]).astype(np.int64)
    n, L = Xt.shape[:2]
    U = torch.empty((n, L, max(int(offs[-1]), 1)), dtype=torch.float64, device=Xt.device)
    if n and L:
        for st, o in zip(slots, offs[:-1]):
            _transform_into(st, Xt, U, int(o))
    return U, offs


def _batch3(X, dev):
    Xt, was_np = _as_tensor(X, dev)
    if Xt.ndim != 3:
        raise ValueError(f"expected an (N, L, d) batch, got shape {tuple(Xt.shape)}")
    return Xt, was_np


def rfsf_exact_gram(state, X, Y=None, normalize: bool = False, counters=None, *, device=None):
    """Exact Gram of a fitted rfsf_full map (features.py:446-475), float64 on
    the device. Numpy in, numpy out; torch in, torch (device) out."""
    cfg = state.config
    if cfg.variant != "rfsf_full":
        raise ValueError(f"exact Gram factorization applies to rfsf_full, not {cfg.variant!r}")
    if counters is None:
        counters = ResourceCounters()
    dev = _device(device)
    Xt, was_np = _batch3(X, dev)
    sym = Y is None
    Yt = Xt if sym else _batch3(Y, dev)[0]
    M = int(cfg.n_levels)
    nx, lx = Xt.shape[:2]
    ny, ly = Yt.shape[:2]
    if M == 0:  # only the constant level (features.py:409-410)
        K = torch.ones((nx, ny), dtype=torch.float64, device=dev)
        return K.cpu().numpy() if was_np else K
    p = int(cfg.effective_order)
    diff = 1 if cfg.difference else 0
    lib = _native.load()
    UX, offs = _lift(state, Xt)
    UY = UX if sym else _lift(state, Yt)[0]
    W = UX.shape[-1]
    offs_c = (ctypes.c_int64 * (M + 1))(*[int(o) for o in offs])
    for st in state.slot_states:
        counters.add_flops(_transform_flops(st, nx * lx) + (0 if sym else _transform_flops(st, ny * ly)))
        counters.add_flops(nx * ny * lx * ly * int(st.out_dim))
    K = torch.zeros((nx, ny), dtype=torch.float64, device=dev)
    if nx == 0 or ny == 0:
        return K.cpu().numpy() if was_np else K
    norm = 1 if normalize else 0
    dx = dy = None
    if normalize:
        dx = _lifted_self(lib, UX, offs_c, M, p, diff)
        dy = dx if sym else _lifted_self(lib, UY, offs_c, M, p, diff)
    buf, nb = _workspace(lib.sk_lifted_gram_workspace_bytes(nx, lx, ny, ly, M, p, diff), dev)
    with torch.cuda.device(dev):
        rc = lib.sk_lifted_gram(UX.data_ptr(), nx, lx, UY.data_ptr(), ny, ly, W, offs_c, M, p,
                                diff, norm, int(sym), 0, nx, ctypes_ptr(dx), ctypes_ptr(dy),
                                K.data_ptr(), ny, None, ctypes_ptr(buf), nb, _stream(dev))
    _native.check(rc, "sk_lifted_gram")
    T1 = max(lx - 1, 0) if diff else lx
    T2 = max(ly - 1, 0) if diff else ly
    counters.add_flops(dp_flops(nx * ny, T1, T2, 0, M, p, False))
    counters.observe_bytes(8 * M * nx * ny * T1 * T2)
    return K.cpu().numpy() if was_np else K


def _lifted_self(lib, U: torch.Tensor, offs_c, M: int, p: int, diff: int) -> torch.Tensor:
    """Self level values (_lifted_self_levels, features.py:427-443), (n, M+1)."""
    n, L, W = U.shape
    out = torch.zeros((n, M + 1), dtype=torch.float64, device=U.device)
    if n == 0:
        return out
    # ny = 1, ly = L: the per-sequence slot Grams of sk_lifted_self_levels
    buf, nb = _workspace(lib.sk_lifted_gram_workspace_bytes(n, L, 1, L, M, p, diff), U.device)
    with torch.cuda.device(U.device):
        rc = lib.sk_lifted_self_levels(U.data_ptr(), n, L, W, offs_c, M, p, diff, out.data_ptr(),
                                       ctypes_ptr(buf), nb, _stream(U.device))
    _native.check(rc, "sk_lifted_self_levels")
    return out
