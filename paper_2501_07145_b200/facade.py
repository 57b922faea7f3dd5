"""KSig-style scikit-learn API (paper).

    K = SignatureKernel(n_levels=5, order=1, normalize=True, static_kernel=RBFKernel())
    K(X, Y)            # (N, N') Gram            -> sig_kernel_gram(X, Y, cfg)
    K(X)               # symmetric K(X, X)       -> sig_kernel_gram(X, None, cfg)
    K(X, diag=True)    # (N,) values k(x_i, x_i)

Mapping onto the reference's KernelConfig (kernels.py:59-91):
n_levels -> n_levels, order -> order (clamped by effective_order),
normalize=True -> normalization="levelwise" ("individually normalizes
signature levels"), difference -> difference,
static_kernel -> StaticKernelSpec (static/kernels.py:39-53).
"""

from __future__ import annotations

import numpy as np
import torch

from .config import KernelConfig, StaticKernelSpec
from .kernels import _batch_points, _device, self_levels, sig_kernel_gram

__all__ = ["StaticKernel", "LinearKernel", "PolynomialKernel", "RBFKernel", "Matern12Kernel",
           "Matern32Kernel", "Matern52Kernel", "RationalQuadraticKernel", "SignatureKernel"]


class StaticKernel:
    """A static kernel on R^d (base class of the KSig static kernels)."""

    spec: StaticKernelSpec

    def __repr__(self) -> str:
        return f"{type(self).__name__}({self.spec})"


class LinearKernel(StaticKernel):
    def __init__(self, scale: float = 1.0):
        self.spec = StaticKernelSpec(kind="linear", scale=scale)


class PolynomialKernel(StaticKernel):
    def __init__(self, degree: int = 3, gamma: float = 1.0, scale: float = 1.0):
        self.spec = StaticKernelSpec(kind="polynomial", degree=degree, gamma=gamma, scale=scale)


class RBFKernel(StaticKernel):
    def __init__(self, bandwidth: float = 1.0):
        self.spec = StaticKernelSpec(kind="rbf", bandwidth=bandwidth)


class Matern12Kernel(StaticKernel):
    def __init__(self, bandwidth: float = 1.0):
        self.spec = StaticKernelSpec(kind="matern12", bandwidth=bandwidth)


class Matern32Kernel(StaticKernel):
    def __init__(self, bandwidth: float = 1.0):
        self.spec = StaticKernelSpec(kind="matern32", bandwidth=bandwidth)


class Matern52Kernel(StaticKernel):
    def __init__(self, bandwidth: float = 1.0):
        self.spec = StaticKernelSpec(kind="matern52", bandwidth=bandwidth)


class RationalQuadraticKernel(StaticKernel):
    def __init__(self, bandwidth: float = 1.0, alpha: float = 1.0):
        self.spec = StaticKernelSpec(kind="rational_quadratic", bandwidth=bandwidth, alpha=alpha)


class SignatureKernel:
    """Truncated signature kernel, callable as K(X, Y) / K(X) / K(X, diag=True)."""

    def __init__(self, n_levels: int = 5, order: int | None = 1, normalize: bool = True,
                 difference: bool = True, static_kernel: StaticKernel | None = None,
                 normalization: str | None = None, precision: str = "fp32", device=None,
                 cuda_graph: bool | str = "auto"):
        static_kernel = static_kernel if static_kernel is not None else RBFKernel()
        if normalization is None:
            normalization = "levelwise" if normalize else "none"
        self.static_kernel = static_kernel
        self.config = KernelConfig(static=static_kernel.spec, n_levels=n_levels, order=order,
                                   difference=difference, normalization=normalization)
        self.precision = precision
        self.device = device
        # cuda_graph=True: repeated calls with the same shapes replay a captured
        # CUDA graph (plan.GramPlan) instead of re-issuing launches from Python;
        # "auto" (default): only for launch-bound calls — arrays/tensors whose
        # Gram has at most GRAPH_CELLS cells (N N' L L'), where host work
        # dominates (c1: 0.15 ms of kernels per call)
        if cuda_graph not in (True, False, "auto"):
            raise ValueError(f"cuda_graph must be True, False or 'auto', got {cuda_graph!r}")
        self.cuda_graph = cuda_graph
        self._plans = {}

    @property
    def n_levels(self) -> int:
        return self.config.n_levels

    @property
    def order(self) -> int:
        return self.config.effective_order

    @property
    def normalize(self) -> bool:
        return self.config.normalization != "none"

    def __call__(self, X, Y=None, diag: bool = False):
        if diag:
            return self.diag(X)
        if self._use_graph(X, Y):
            from .plan import GramPlan
            key = (tuple(X.shape), None if Y is None else tuple(Y.shape))
            plan = self._plans.get(key)
            if plan is None:
                if len(self._plans) >= self.MAX_PLANS:  # oldest shape out
                    self._plans.pop(next(iter(self._plans)))
                plan = self._plans[key] = GramPlan(self.config, key[0], key[1],
                                                   precision=self.precision, device=self.device)
            return plan(X, Y)
        return sig_kernel_gram(X, Y, cfg=self.config, precision=self.precision,
                               device=self.device)

    GRAPH_CELLS = 1 << 28
    MAX_PLANS = 8

    def _use_graph(self, X, Y) -> bool:
        if self.cuda_graph is not True and self.cuda_graph != "auto":
            return False
        if self.cuda_graph is True:
            return True
        arr = (np.ndarray, torch.Tensor)
        if not isinstance(X, arr) or (Y is not None and not isinstance(Y, arr)):
            return False
        if X.ndim != 3 or (Y is not None and Y.ndim != 3) or not torch.cuda.is_available():
            return False
        dev = _device(self.device)
        for t in (X, Y):
            if isinstance(t, torch.Tensor) and (not t.is_cuda or t.device != dev
                                                or t.dtype != torch.float64):
                return False
        nx, lx = int(X.shape[0]), int(X.shape[1])
        ny, ly = (nx, lx) if Y is None else (int(Y.shape[0]), int(Y.shape[1]))
        if min(nx, ny) < 1 or min(lx, ly) < 2:
            return False
        return nx * ny * lx * ly <= self.GRAPH_CELLS

    def diag(self, X):
        """k(x_i, x_i) for every sequence (the diagonal of K(X)).

        Unnormalised: sum of self levels (kernels.py:589-590). Levelwise:
        (1/(M+1)) * #{m : k_m(x,x) > 0} (kernels.py:510-516 with x = y).
        Global: 1 (kernels.py:519-527; raises NumericError if k(x,x) <= 0).
        """
        dev = X.device if isinstance(X, torch.Tensor) and X.is_cuda else _device(self.device)
        Xt, was_np = _batch_points(X, dev)
        lv = self_levels(Xt, self.config, self.precision)
        norm = self.config.normalization
        if norm == "none":
            out = lv.sum(dim=-1)
        elif norm == "levelwise":
            out = (lv > 0).to(torch.float64).sum(dim=-1) / (self.config.n_levels + 1)
        else:
            from .kernels import _check_global
            _check_global(lv, lv)
            tot = lv.sum(dim=-1)
            out = tot / torch.sqrt(tot * tot)
        return out.cpu().numpy() if was_np else out

    def __repr__(self) -> str:
        c = self.config
        return (f"SignatureKernel(n_levels={c.n_levels}, order={c.order}, "
                f"normalization={c.normalization!r}, difference={c.difference}, "
                f"static_kernel={self.static_kernel!r})")
