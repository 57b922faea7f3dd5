"""Analytic resource accounting (reference: sigkern/utils.py:10-40).

`flops` counts multiply-adds exactly as the reference's counters do for the
same work (so `counters=` callers see the same totals); `peak_bytes` is the
analytic high-water mark of this implementation's device buffers, which is
linear in the sequence length (the reference's is quadratic, kernels.py:443).
"""

from __future__ import annotations

__all__ = ["ResourceCounters"]


class ResourceCounters:
    __slots__ = ("flops", "peak_bytes")

    def __init__(self):
        self.flops = 0
        self.peak_bytes = 0

    def add_flops(self, n) -> None:
        self.flops += int(n)

    def observe_bytes(self, n) -> None:
        self.peak_bytes = max(self.peak_bytes, int(n))

    def merge(self, other: "ResourceCounters") -> None:
        self.flops += other.flops
        self.peak_bytes = max(self.peak_bytes, other.peak_bytes)

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
