"""CUDA-graph plans for launch-bound, repeated fixed-shape Gram calls.

A small Gram (BASELINE c1: 64 x 64 sequences of 50 points) is ~30 us of
kernel time inside ~400 us of host work per `sig_kernel_gram` call (argument
checks, workspace and output allocation, config marshalling, ctypes, 6
launches). `GramPlan` records the whole device sequence of one call — the
self-level launches for normalisation and the `sk_gram` launches — once into
a CUDA graph over static input/output buffers, and every call then costs one
copy into the static inputs, one graph replay and one fused validity check.

Semantics match `sig_kernel_gram` (same kernels, same arithmetic, same
errors): non-finite inputs raise ValueError("... non-finite ...") and a
non-positive self-kernel under global normalisation raises NumericError, both
checked after the replay with a single device-to-host read.
"""

from __future__ import annotations

import numpy as np
import torch

from .config import KernelConfig
from .errors import NumericError
from .kernels import _device, _self_levels_t, gram_block

__all__ = ["GramPlan"]


class GramPlan:
    """K(X, Y) (or K(X) if `y_shape` is None) for inputs of fixed shapes, replayed
    from a captured CUDA graph."""

    def __init__(self, cfg: KernelConfig, x_shape, y_shape=None, precision: str = "fp32",
                 device=None):
        self.cfg = cfg
        self.precision = precision
        self.dev = _device(device)
        self.x_shape = tuple(int(v) for v in x_shape)
        self.y_shape = None if y_shape is None else tuple(int(v) for v in y_shape)
        if len(self.x_shape) != 3 or (self.y_shape is not None and len(self.y_shape) != 3):
            raise ValueError("expected (N, L, d) shapes")
        if self.y_shape is not None and self.y_shape[2] != self.x_shape[2]:
            raise ValueError(f"channel mismatch: d={self.x_shape[2]} vs d={self.y_shape[2]}")
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.X = torch.zeros(self.x_shape, **f64)
        self.Y = None if self.y_shape is None else torch.zeros(self.y_shape, **f64)
        # warm up eagerly on a side stream (loads the library, sets kernel
        # attributes, primes the allocator), then capture
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self._run()
        torch.cuda.current_stream(self.dev).wait_stream(side)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.K, self._ok = self._run()
        self.launches = None  # filled lazily by tools that inspect the graph

    def _run(self):
        cfg, prec = self.cfg, self.precision
        dx = dy = None
        if cfg.normalization != "none":
            dx = _self_levels_t(self.X, cfg, prec)
            dy = dx if self.Y is None else _self_levels_t(self.Y, cfg, prec)
        K, _ = gram_block(self.X, self.Y, cfg, precision=prec, diag_x=dx, diag_y=dy,
                          check_global=False)
        # validity flags, read after the replay: inputs finite, global self-kernels > 0
        ok = torch.isfinite(self.X).all().reshape(1)
        if self.Y is not None:
            ok = ok & torch.isfinite(self.Y).all().reshape(1)
        if cfg.normalization == "global":
            ok = torch.cat([ok, (dx.sum(-1) > 0).all().reshape(1),
                            (dy.sum(-1) > 0).all().reshape(1)])
        return K, ok

    def __call__(self, X, Y=None):
        was_np = not isinstance(X, torch.Tensor)
        for src, dst, shape, what in ((X, self.X, self.x_shape, "X"),
                                      (Y, self.Y, self.y_shape, "Y")):
            if dst is None:
                if src is not None:
                    raise ValueError("this plan computes K(X); build one with y_shape for K(X, Y)")
                continue
            t = src if isinstance(src, torch.Tensor) else torch.from_numpy(np.asarray(src, np.float64))
            if tuple(t.shape) != shape:
                raise ValueError(f"{what} has shape {tuple(t.shape)}, plan was built for {shape}")
            dst.copy_(t, non_blocking=True)
        self.graph.replay()
        ok = self._ok.cpu()
        if not bool(ok[0]):
            raise ValueError("sequence batch contains non-finite values")
        if ok.numel() > 1 and not bool(ok[1:].all()):
            self._raise_global()
        return self.K.cpu().numpy() if was_np else self.K.clone()

    def _raise_global(self):
        # reproduce the reference's message (kernels.py:519-527)
        cfg, prec = self.cfg, self.precision
        dx = _self_levels_t(self.X, cfg, prec)
        dy = dx if self.Y is None else _self_levels_t(self.Y, cfg, prec)
        for s in (dx.sum(-1), dy.sum(-1)):
            bad = torch.nonzero(s <= 0).flatten()
            if bad.numel():
                raise NumericError(
                    f"global normalization undefined: non-positive self-kernel for "
                    f"input sequence index {int(bad[0])}")
