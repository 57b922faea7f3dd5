"""Kernel configuration (reference: static/kernels.py:39-65, kernels.py:59-111).

Same fields, defaults, validation rules and messages as the reference's
frozen dataclasses, so `KernelConfig`/`StaticKernelSpec` objects are
interchangeable at the boundary.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["KERNEL_KINDS", "NORMALIZATIONS", "StaticKernelSpec", "KernelConfig", "LevelValues"]

KERNEL_KINDS = ("linear", "polynomial", "rbf", "matern12", "matern32", "matern52",
                "rational_quadratic")  # static/kernels.py:25-33
NORMALIZATIONS = ("none", "levelwise", "global")  # kernels.py:52


@dataclass(frozen=True)
class StaticKernelSpec:
    """Static (pointwise) kernel and its parameters (static/kernels.py:39-65)."""

    kind: str = "rbf"
    scale: float = 1.0
    degree: int = 3
    gamma: float = 1.0
    bandwidth: float = 1.0
    alpha: float = 1.0

    def __post_init__(self):
        if self.kind not in KERNEL_KINDS:
            raise ValueError(f"unknown kernel kind {self.kind!r}; choose from {KERNEL_KINDS}")
        if not self.scale > 0:
            raise ValueError(f"scale must be positive, got {self.scale}")
        if not (isinstance(self.degree, (int, np.integer)) and self.degree >= 1):
            raise ValueError(f"degree must be a positive integer, got {self.degree}")
        if not self.bandwidth > 0:
            raise ValueError(f"bandwidth must be positive, got {self.bandwidth}")
        if not self.alpha > 0:
            raise ValueError(f"alpha must be positive, got {self.alpha}")


@dataclass(frozen=True)
class KernelConfig:
    """Truncation level M, order p, differencing and normalisation (kernels.py:59-91)."""

    static: StaticKernelSpec = field(default_factory=StaticKernelSpec)
    n_levels: int = 5
    order: int | None = 1
    difference: bool = True
    normalization: str = "none"

    def __post_init__(self):
        if not (isinstance(self.n_levels, (int, np.integer)) and self.n_levels >= 0):
            raise ValueError(f"n_levels must be a non-negative integer, got {self.n_levels}")
        if self.order is not None and not (
                isinstance(self.order, (int, np.integer)) and self.order >= 1):
            raise ValueError(f"order must be a positive integer or None, got {self.order}")
        if self.normalization not in NORMALIZATIONS:
            raise ValueError(
                f"normalization must be one of {NORMALIZATIONS}, got {self.normalization!r}")

    @property
    def effective_order(self) -> int:
        """kernels.py:85-91: 1 if M = 0, M if order is None, else min(order, M)."""
        if self.n_levels == 0:
            return 1
        if self.order is None:
            return int(self.n_levels)
        return min(int(self.order), int(self.n_levels))


@dataclass
class LevelValues:
    """Per-level kernel values k_0..k_M (kernels.py:94-111)."""

    values: np.ndarray

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)

    @property
    def n_levels(self) -> int:
        return self.values.shape[-1] - 1

    def total(self) -> float:
        return float(self.values.sum())

    def __getitem__(self, m):
        return self.values[m]
