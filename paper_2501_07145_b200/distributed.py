"""Multi-GPU Gram: one process per GPU, rows of K sharded across ranks.

The reference parallelises over fixed pair tiles on a host thread pool
(kernels.py:437-473 -> utils.py:43-57); every Gram entry is independent
(SPEC.md:335). Here each rank evaluates a contiguous block of rows of K on
its own GPU (the `sk_gram` row range), then one NCCL collective over
NVLink/NVSwitch assembles the finished rows on every rank:

* cross K(X, Y): equal row blocks, `all_gather_into_tensor` of the
  (padded) blocks;
* symmetric K(X): the rows are cut into 2*world equal blocks and rank r
  evaluates the upper-triangle pairs of blocks r and 2*world-1-r (the same
  number of pairs on every rank); one `all_gather_into_tensor` of those rows
  (half the bytes of an all-reduce of the full matrix) and a bitwise mirror
  of the upper triangle assemble K.

`compute` is injectable so the host logic can be exercised with the gloo
backend on CPU (tests/test_distributed.py); the default computes on the
rank's GPU through the C ABI.
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist

from .config import KernelConfig

__all__ = ["row_blocks", "triangle_row_blocks", "paired_row_blocks", "sharded_gram"]


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


def paired_row_blocks(n: int, world: int) -> list[tuple[tuple[int, int], tuple[int, int]]]:
    """Rank r's two row blocks (r and 2*world-1-r of 2*world equal blocks): the
    upper-triangle pair counts of the two add up to the same total on every rank."""
    b = max(1, math.ceil(n / (2 * world))) if n else 0
    blk = [(min(k * b, n), min((k + 1) * b, n)) for k in range(2 * world)]
    return [(blk[r], blk[2 * world - 1 - r]) for r in range(world)]


def _all_gather(out: torch.Tensor, inp: torch.Tensor, group) -> None:
    """all_gather_into_tensor; a gloo group (CPU tests, or ranks sharing one GPU)
    takes host copies of device tensors."""
    if inp.is_cuda and dist.get_backend(group) == "gloo":
        host = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(host, inp.cpu(), group=group)
        out.copy_(host)
        return
    dist.all_gather_into_tensor(out, inp, group=group)


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
        blocks = paired_row_blocks(nx, world)
        b = blocks[0][0][1] - blocks[0][0][0]  # rows per block (the last ones may be short)
        # symmetric sk_gram calls write their rows i <= j and the mirror of
        # them into a full local matrix; only this rank's rows are sent
        K_loc = torch.zeros((nx, nx), dtype=torch.float64, device=X.device)
        send = torch.zeros((2 * b, nx), dtype=torch.float64, device=X.device)
        for k, (a0, a1) in enumerate(blocks[rank]):
            if a1 > a0:
                compute(X, None, cfg, a0, a1, precision, K_loc)
                send[k * b:k * b + a1 - a0] = K_loc[a0:a1]
        del K_loc
        got = torch.empty((world * 2 * b, nx), dtype=torch.float64, device=X.device)
        _all_gather(got, send, group)
        K = torch.empty((nx, nx), dtype=torch.float64, device=X.device)
        for r, rb in enumerate(blocks):
            for k, (a0, a1) in enumerate(rb):
                if a1 > a0:
                    K[a0:a1] = got[(2 * r + k) * b:(2 * r + k) * b + a1 - a0]
        del got
        # rows hold the pairs i <= j; the lower triangle is their mirror (bitwise)
        upper = torch.ones((nx, nx), dtype=torch.bool, device=X.device).triu_()
        return torch.where(upper, K, K.T)
    ny = Y.shape[0]
    blocks = row_blocks(nx, world)
    b = blocks[0][1] - blocks[0][0]
    r0, r1 = blocks[rank]
    local = torch.zeros((b, ny), dtype=torch.float64, device=X.device)
    if r1 > r0:
        local[: r1 - r0] = compute(X, Y, cfg, r0, r1, precision, None)
    out = torch.empty((b * world, ny), dtype=torch.float64, device=X.device)
    _all_gather(out, local, group)
    return out[:nx]
