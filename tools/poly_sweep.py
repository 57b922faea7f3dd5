"""Polynomial kind on the fused FP32 path: max relative error vs float64 per
n_levels over random cases (development)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import execution_path, gram_block  # noqa: E402

worst = {}
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 400):
    r = np.random.default_rng(5000 + seed)
    M = int(r.integers(1, 9))
    p = 1 if r.random() < 0.6 else int(r.integers(1, M + 1))
    deg = int(r.integers(1, 5))
    norm = ("none", "levelwise", "global")[int(r.integers(0, 3))]
    d = int((2, 3, 5, 8, 13, 16)[int(r.integers(0, 6))])
    lx, ly = int(r.integers(2, 90)), int(r.integers(2, 90))
    kw = dict(scale=float(r.uniform(0.3, 1.5)), degree=deg, gamma=float(r.uniform(0.0, 1.5)))
    cfg = KernelConfig(static=StaticKernelSpec(kind="polynomial", **kw), n_levels=M, order=p,
                       normalization=norm)
    if execution_path(lx, ly, d, cfg) != "fused":
        continue
    X = torch.from_numpy(gen_brownian(6, lx, d, SeedStream(seed, ("x",))).data).cuda()
    Y = torch.from_numpy(gen_brownian(5, ly, d, SeedStream(seed, ("y",))).data).cuda()
    try:
        K = gram_block(X, Y, cfg)[0].cpu().numpy()
        K6 = gram_block(X, Y, cfg, precision="fp64")[0].cpu().numpy()
    except Exception as e:  # noqa: BLE001 (global normalisation of a non-positive self kernel)
        continue
    err = float((np.abs(K - K6) / np.maximum(np.abs(K6), 1e-12 * np.abs(K6).max())).max())
    tol = 1e-4 if norm == "none" else 1e-5
    key = (M, deg)
    if err / tol > worst.get(key, (0, None))[0]:
        worst[key] = (err / tol, (seed, M, p, deg, norm, d, lx, ly, err))
for k in sorted(worst):
    print(k, "worst err/tol %.3f" % worst[k][0], worst[k][1])
