"""Per-level FP32 vs float64 errors of one fuzz seed's worst entry (development)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_gpu_fuzz as F  # noqa: E402
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, _native, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import gram_block  # noqa: E402

for seed in map(int, sys.argv[1:]):
    kind, kw, M, order, norm, diff, d, lx, ly, sym = F._case(seed)
    X = gen_brownian(5, lx, d, SeedStream(seed, ("x",))).data
    Y = None if sym else gen_brownian(4, ly, d, SeedStream(seed, ("y",))).data
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=order,
                       difference=diff, normalization="none")
    Xt = torch.from_numpy(X).cuda()
    Yt = None if Y is None else torch.from_numpy(Y).cuda()
    K0, lv0 = gram_block(Xt, Yt, cfg, want_levels=True, flags=_native.SK_FLAG_NO_FIXUP)
    K1, lv1 = gram_block(Xt, Yt, cfg, want_levels=True)
    K6, lv6 = gram_block(Xt, Yt, cfg, want_levels=True, precision="fp64")
    K0, K1, K6 = K0.cpu().numpy(), K1.cpu().numpy(), K6.cpu().numpy()
    lv0, lv6 = lv0.cpu().numpy(), lv6.cpu().numpy()
    e = np.abs(K1 - K6) / np.abs(K6)
    i, j = np.unravel_index(np.argmax(e), e.shape)
    print(f"seed {seed} {kind} {kw} M={M} p={order} d={d} L={lx},{ly}: worst ({i},{j}) certified err {e[i, j]:.2e}"
          f" raw err {abs(K0[i, j] - K6[i, j]) / abs(K6[i, j]):.2e} K={K6[i, j]:.4e} sum|k_m|={np.abs(lv6[i, j]).sum():.4e}")
    for m in range(M + 1):
        print(f"   level {m}: f64 {lv6[i, j, m]: .6e}  fp32 {lv0[i, j, m]: .6e}  rel {abs(lv0[i, j, m] - lv6[i, j, m]) / max(abs(lv6[i, j, m]), 1e-300):.2e}")
