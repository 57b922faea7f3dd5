"""Certification diagnostics (development tool): for a config's shapes, how
many entries the FP32 epilogue flags (SK_FLAG_NO_FIXUP), and the realised
level-1 deviation of the FP32 levels from the exact telescoped value.

    python tools/diag_cert.py <name> <n>     (name from bench.CONFIGS)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import sigkern_oracle as O  # noqa: E402
from paper_2501_07145_b200 import SeedStream, _native, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import _self_levels_t, gram_block  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
N, L, d, M, p, kind, norm, sym, _ = bench.CONFIGS[name]
cfg = bench.kernel_config(name)
X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
F = _native.SK_FLAG_NO_FIXUP
dx = dy = None
if norm != "none":
    dx = _self_levels_t(X, cfg, "fp32", flags=F)
    dy = _self_levels_t(Y, cfg, "fp32", flags=F)
K, lv = gram_block(X, Y, cfg, diag_x=dx, diag_y=dy, flags=F, want_levels=True)
print(name, "n", n, "flagged by the epilogue:", int(torch.isnan(K).sum()), "of", K.numel())
Xh, Yh = X.cpu().numpy(), Y.cpu().numpy()
sp = O.static_params(kind)
G = O.point_gram(sp, Xh[:, None, [0, -1]], Yh[None, :, [0, -1]])  # corners
k1 = G[..., 1, 1] - G[..., 0, 1] - G[..., 1, 0] + G[..., 0, 0]
lv = lv.cpu().numpy()
dev = np.abs(lv[..., 1] - k1)
Kc = K.cpu().numpy()
print("level-1 |FP32 - exact|: median %.2e max %.2e; relative to |K|: median %.2e max %.2e" % (
    np.median(dev), dev.max(), np.median(dev / np.abs(Kc)), np.nanmax(dev / np.abs(Kc))))
print("K: min |K| %.3e median %.3e" % (np.nanmin(np.abs(Kc)), np.nanmedian(np.abs(Kc))))
s = np.abs(lv).sum(-1)
print("|K| / sum|k_m|: min %.3e median %.3e" % (np.nanmin(np.abs(Kc) / s), np.nanmedian(np.abs(Kc) / s)))
r = np.abs(lv.sum(-1)) / s  # from the level values (K itself is NaN where flagged)
for t in (1e-2, 3e-3, 1e-3, 3e-4):
    print("fraction with |K| < %.0e sum|k_m|: %.2e" % (t, float(np.mean(r < t))))
# FP32 error (after the exact-level-1 correction) against float64, bucketed by
# the cancellation ratio |K| / sum_m |k_m| the certification rule uses
if norm == "none":
    K64 = gram_block(X, Y, cfg, precision="fp64")[0].cpu().numpy()
    K32c = lv.sum(-1) - lv[..., 1] + k1
    err = np.abs(K32c - K64) / np.abs(K64)
    r = np.abs(lv.sum(-1)) / s
    for lo, hi in ((0, 1e-4), (1e-4, 3e-4), (3e-4, 1e-3), (1e-3, 1e-2), (1e-2, 10)):
        m = (r >= lo) & (r < hi)
        if m.any():
            print("ratio [%.0e, %.0e): %d entries, FP32 rel err max %.2e median %.2e"
                  % (lo, hi, int(m.sum()), err[m].max(), np.median(err[m])))
