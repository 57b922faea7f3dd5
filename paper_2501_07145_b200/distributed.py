"""Multi-GPU Gram: one process per GPU, rows of K sharded across ranks.

The reference parallelises over fixed pair tiles on a host thread pool
(kernels.py:437-473 -> utils.py:43-57); every Gram entry is independent
(SPEC.md:335). Here each rank evaluates a contiguous block of rows of K on
its own GPU (the `sk_gram` row range), then one NCCL collective over
NVLink/NVSwitch assembles the finished rows on every rank:

* cross K(X, Y): equal row blocks, `all_gather_into_tensor` of the
  (padded) blocks;
* symmetric K(X): rows are split so every rank gets the same number of
  upper-triangle pairs; each rank writes its triangle rows and their mirror
  into a zeroed full matrix and one `all_reduce(SUM)` assembles K (every
  entry has exactly one non-zero contributor, so the sum is exact).

`compute` is injectable so the host logic can be exercised with the gloo
backend on CPU (tests/test_distributed.py); the default computes on the
rank's GPU through the C ABI.
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from .config import KernelConfig

__all__ = ["row_blocks", "triangle_row_blocks", "sharded_gram"]


def row_blocks(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, equal-size (last may be short) row blocks of ceil(n/world) rows."""
    b = max(1, math.ceil(n / world)) if n else 0
    return [(min(r * b, n), min((r + 1) * b, n)) for r in range(world)]


def triangle_row_blocks(n: int, world: int) -> list[tuple[int, int]]:
    """Row blocks with (nearly) equal counts of upper-triangle pairs (i <= j)."""
    total = n * (n + 1) // 2
    bounds = [0]
    acc = 0
    i = 0
    for r in range(1, world):
        target = total * r / world
        while i < n and acc + (n - i) <= target:
            acc += n - i
            i += 1
        bounds.append(i)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def _default_compute(X, Y, cfg, r0, r1, precision, K_full=None):
    from .kernels import gram_block
    K, _ = gram_block(X, Y, cfg, row_begin=r0, row_end=r1, precision=precision, K=K_full)
    return K


def sharded_gram(X: torch.Tensor, Y: torch.Tensor | None, cfg: KernelConfig,
                 precision: str = "fp32", group=None, compute=None) -> torch.Tensor:
    """Full K on every rank of `group` (X, Y already on this rank's device).

    compute(X, Y, cfg, r0, r1, precision, K_full) -> rows [r0, r1) of K
    (cross) or fills K_full in place (symmetric).
    """
    compute = compute or _default_compute
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nx = X.shape[0]
    if Y is None:
        r0, r1 = triangle_row_blocks(nx, world)[rank]
        K = torch.zeros((nx, nx), dtype=torch.float64, device=X.device)
        compute(X, None, cfg, r0, r1, precision, K)
        dist.all_reduce(K, op=dist.ReduceOp.SUM, group=group)
        return K
    ny = Y.shape[0]
    blocks = row_blocks(nx, world)
    b = blocks[0][1] - blocks[0][0]
    r0, r1 = blocks[rank]
    local = torch.zeros((b, ny), dtype=torch.float64, device=X.device)
    if r1 > r0:
        local[: r1 - r0] = compute(X, Y, cfg, r0, r1, precision, None)
    out = torch.empty((b * world, ny), dtype=torch.float64, device=X.device)
    dist.all_gather_into_tensor(out, local, group=group)
    return out[:nx]
