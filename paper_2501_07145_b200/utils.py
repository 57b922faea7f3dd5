"""Analytic resource accounting (reference: sigkern/utils.py:10-40).

`flops` and `peak_bytes` are the reference's analytic model of the same
call, reproduced term for term (the tile structure of kernels.py:437-473 and
476-507, the DP counts of kernels.py:170-200, increment_tensor's of
:273-280, _pde_stream's of :358-399), so `counters=` callers — the bench
records, the acceptance criteria's scaling checks — see the reference's
numbers. The device's own footprint (linear in the sequence length: the
fused kernels never materialise the L x L' grid) is kept separately in
`device_bytes`.
"""

from __future__ import annotations

import math

__all__ = ["ResourceCounters", "gram_counts"]

_DP_STATE_ARRAYS = 6  # kernels.py:56


class ResourceCounters:
    __slots__ = ("flops", "peak_bytes", "device_bytes")

    def __init__(self):
        self.flops = 0
        self.peak_bytes = 0
        self.device_bytes = 0

    def add_flops(self, n) -> None:
        self.flops += int(n)

    def observe_bytes(self, n) -> None:
        self.peak_bytes = max(self.peak_bytes, int(n))

    def observe_device_bytes(self, n) -> None:
        self.device_bytes = max(self.device_bytes, int(n))

    def merge(self, other: "ResourceCounters") -> None:
        self.flops += other.flops
        self.peak_bytes = max(self.peak_bytes, other.peak_bytes)
        self.device_bytes = max(self.device_bytes, getattr(other, "device_bytes", 0))

    def __repr__(self) -> str:
        return f"ResourceCounters(flops={self.flops}, peak_bytes={self.peak_bytes})"


def dp_flops(pairs: int, T1: int, T2: int, d: int, M: int, p: int, difference: bool) -> int:
    """Multiply-adds the reference counts for `pairs` pair-DPs.

    increment_tensor: G.size * d + 3 * T1 * T2 (kernels.py:273-280);
    sig_levels_dp: kernels.py:178-199.
    """
    L1 = T1 + 1 if difference else T1
    L2 = T2 + 1 if difference else T2
    inc = L1 * L2 * d + (3 * T1 * T2 if difference else 0)
    cell = T1 * T2
    lv = 0
    if M >= 1 and cell > 0:
        lv = cell
        for _ in range(2, M + 1):
            lv += (p * p + 3) * cell
            if p > 1:
                lv += 2 * p * p * cell + (p - 1) * 4 * cell + (p - 1) ** 2 * 2 * cell
            lv += p * p * cell
    return pairs * (inc + lv)


def _tiles(nx: int, ny: int, b: int, symmetric: bool):
    """The reference's pair tiles (kernels.py:446-454, 480-488)."""
    rows = [(i, min(i + b, nx)) for i in range(0, nx, b)]
    cols = [(j, min(j + b, ny)) for j in range(0, ny, b)]
    return [(i0, i1, j0, j1) for bi, (i0, i1) in enumerate(rows)
            for bj, (j0, j1) in enumerate(cols) if not (symmetric and bj < bi)]


def _increment_counts(c, lead: int, L1: int, L2: int, d: int, difference: bool) -> None:
    # kernels.py:273-280
    c.add_flops(lead * L1 * L2 * d)
    if difference and L1 >= 2 and L2 >= 2:
        c.add_flops(3 * (L2 - 1) * (L1 - 1) * lead)


def _levels_counts(c, lead: int, T1: int, T2: int, M: int, p: int) -> None:
    # kernels.py:170-200 (early return before any count when the grid is empty)
    if M == 0 or T1 == 0 or T2 == 0:
        return
    c.add_flops(dp_flops(lead, T1, T2, 0, M, p, False))
    c.observe_bytes((2 * p * p + _DP_STATE_ARRAYS) * lead * T1 * T2 * 8)


def _pde_counts(c, lead: int, Lx: int, Ly: int, d: int, difference: bool) -> None:
    # _pde_stream, kernels.py:349-399
    T1, T2 = (Lx - 1, Ly - 1) if difference else (Lx, Ly)
    if difference and (T1 < 1 or T2 < 1):
        return
    c.observe_bytes((6 * lead * (min(T1, T2) + 1) + 2 * lead * (min(T1, T2) + 1) * d) * 8)
    points = (T1 + 1) * (T2 + 1) if difference else T1 * T2
    c.add_flops(lead * points * d + lead * T1 * T2 * 6)


def gram_counts(c, nx: int, lx: int, ny: int, ly: int, d: int, M: int, p: int,
                difference: bool, normalization: str, symmetric: bool, algorithm: str = "dp",
                tile_memory: int = 256 * 2 ** 20) -> None:
    """Add the reference's counts for sig_kernel_gram (kernels.py:530-600)."""
    if algorithm == "pde":
        b = max(1, math.isqrt(max(1, int(tile_memory) // (8 * 8 * (lx + ly)))))
        for i0, i1, j0, j1 in _tiles(nx, ny, b, symmetric):
            local = ResourceCounters()
            _pde_counts(local, (i1 - i0) * (j1 - j0), lx, ly, d, difference)
            c.merge(local)
        if normalization == "global":
            _pde_counts(c, nx, lx, lx, d, difference)
            if not symmetric:
                _pde_counts(c, ny, ly, ly, d, difference)
        return
    T1 = lx - 1 if difference else lx
    T2 = ly - 1 if difference else ly
    T1, T2 = max(T1, 0), max(T2, 0)
    per_pair = 8 * (lx * ly + (2 * p * p + _DP_STATE_ARRAYS) * max(T1 * T2, 1))
    b = max(1, math.isqrt(max(1, int(tile_memory) // per_pair)))
    for i0, i1, j0, j1 in _tiles(nx, ny, b, symmetric):
        local = ResourceCounters()
        tp = (i1 - i0) * (j1 - j0)
        _increment_counts(local, tp, lx, ly, d, difference)
        _levels_counts(local, tp, T1, T2, M, p)
        local.observe_bytes(tp * per_pair)
        c.merge(local)
    if normalization == "none":
        return
    _increment_counts(c, nx, lx, lx, d, difference)
    _levels_counts(c, nx, T1, T1, M, p)
    if not symmetric:
        _increment_counts(c, ny, ly, ly, d, difference)
        _levels_counts(c, ny, T2, T2, M, p)
