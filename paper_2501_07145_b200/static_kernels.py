"""Static-kernel helpers of the reference's `sigkern.static.kernels` that the
Gram path uses: `median_heuristic` (static/kernels.py:165-187), the bandwidth
rule the reference's CLI and benchmarks apply for `bandwidth = median`
(cli.py:72-81, benchmarks.py:180-183).

The pairwise distances run on the GPU (`sk_pairwise_dist`, float64, the
reference's norm-expansion formula); subsampling and the median follow the
reference exactly.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native

__all__ = ["median_heuristic"]


def median_heuristic(X, max_pairs: int = 1_000_000, device=None) -> float:
    """Median pairwise Euclidean distance over a deterministic subsample.

    When the full pair count exceeds max_pairs, an evenly spaced subset of
    rows whose pair count fits the budget is used instead. A zero median
    (all subsampled points equal) falls back to 1.0. (static/kernels.py:165-187)
    """
    from .kernels import _device, _stream
    if isinstance(X, torch.Tensor):
        Xt = X.detach().to(torch.float64)
        Xt = Xt.reshape(1, -1) if Xt.dim() < 2 else Xt
    else:
        Xt = torch.from_numpy(np.atleast_2d(np.asarray(X, dtype=np.float64)))
    n = Xt.shape[0]
    if n < 2:
        raise ValueError(f"median_heuristic needs at least 2 vectors, got {n}")
    if max_pairs < 1:
        raise ValueError(f"max_pairs must be positive, got {max_pairs}")
    if n * (n - 1) // 2 > max_pairs:
        m = int((1.0 + math.sqrt(1.0 + 8.0 * max_pairs)) / 2.0)
        m = max(2, min(n, m))
        idx = np.unique((np.arange(m, dtype=np.int64) * n) // m)
        Xt = Xt[torch.from_numpy(idx).to(Xt.device)]
        n = Xt.shape[0]
    dev = Xt.device if Xt.is_cuda else _device(device)
    Xd = Xt.to(dev).contiguous()
    npairs = n * (n - 1) // 2
    out = torch.empty(npairs, dtype=torch.float64, device=dev)
    lib = _native.load()
    with torch.cuda.device(dev):
        rc = lib.sk_pairwise_dist(Xd.data_ptr(), n, Xd.shape[1], out.data_ptr(), _stream(dev))
    _native.check(rc, "sk_pairwise_dist")
    s = torch.sort(out).values
    mid = npairs // 2
    med = float(s[mid]) if npairs % 2 else float((s[mid - 1] + s[mid]) / 2.0)  # np.median
    return med if med > 0.0 else 1.0
