"""FP32 paths vs float64 over random configurations: worst error / tolerance per
(kind, path, order class, difference, d class) (development; also the case
generator of tests/test_gpu_path_sweep.py).

    python tools/path_sweep.py [cases] [first seed] [long | smallbw]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import execution_path, gram_block  # noqa: E402

KINDS = ("rbf", "linear", "matern12", "matern32", "matern52", "rational_quadratic")


def make_case(seed, long=False, small_bw=False):
    """(cfg, d, lx, ly, description) of sweep case `seed`."""
    r = np.random.default_rng(9000 + seed)
    kind = KINDS[int(r.integers(0, len(KINDS)))]
    M = int(r.integers(1, 9))
    p = 1 if r.random() < 0.4 else int(r.integers(1, M + 1))
    norm = ("none", "levelwise", "global")[int(r.integers(0, 3))]
    diff = bool(r.random() < 0.8)
    d = int((2, 3, 5, 8, 13, 16, 20, 40)[int(r.integers(0, 8))])
    lx, ly = int(r.integers(2, 120)), int(r.integers(2, 120))
    if r.random() < 0.3:
        lx, ly = int(r.integers(6, 30)), int(r.integers(6, 30))
    if long:  # multi-panel rows and long x rings
        lx, ly = int(r.integers(120, 700)), int(r.integers(120, 700))
    kw = {}
    if kind != "linear":
        kw["bandwidth"] = float(r.uniform(0.4, 2.0))
        if small_bw:  # points far apart on the kernel's scale
            kw["bandwidth"] = float(r.uniform(0.05, 0.4))
    else:
        kw["scale"] = float(r.uniform(0.3, 1.5))
    if kind == "rational_quadratic":
        kw["alpha"] = float(r.uniform(0.5, 3.0))
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=p,
                       difference=diff, normalization=norm)
    return cfg, d, lx, ly, (kind, M, p, norm, diff, d, lx, ly)


def run_case(seed, long=False, small_bw=False):
    """(path, error / tolerance, description); path None when the case is not
    on an FP32 path or its global normalisation is undefined."""
    cfg, d, lx, ly, desc = make_case(seed, long, small_bw)
    path = execution_path(lx, ly, d, cfg)
    if path == "fp64":
        return None, 0.0, desc
    X = torch.from_numpy(gen_brownian(6, lx, d, SeedStream(seed, ("x",))).data).cuda()
    Y = torch.from_numpy(gen_brownian(5, ly, d, SeedStream(seed, ("y",))).data).cuda()
    try:
        K = gram_block(X, Y, cfg)[0].cpu().numpy()
        K6 = gram_block(X, Y, cfg, precision="fp64")[0].cpu().numpy()
    except Exception:  # noqa: BLE001 (global normalisation of a non-positive self kernel)
        return None, 0.0, desc
    err = float((np.abs(K - K6) / np.maximum(np.abs(K6), 1e-12 * np.abs(K6).max())).max())
    tol = 1e-4 if cfg.normalization == "none" else 1e-5
    return path, err / tol, desc


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    long = len(sys.argv) > 3 and sys.argv[3] == "long"
    small_bw = len(sys.argv) > 3 and sys.argv[3] == "smallbw"
    worst, n = {}, 0
    for seed in range(first, first + count):
        path, ratio, desc = run_case(seed, long, small_bw)
        if path is None:
            continue
        n += 1
        kind, M, p, norm, diff, d = desc[:6]
        key = (kind if not kind.startswith("matern") else "matern", path,
               "p1" if p == 1 else "p>1", "diff" if diff else "nodiff", "d2" if d == 2 else "d>2")
        if ratio > worst.get(key, (0, None))[0]:
            worst[key] = (ratio, (seed,) + desc)
    print("cases on FP32 paths:", n)
    for k in sorted(worst):
        flag = "  <-- FAIL" if worst[k][0] > 1 else ""
        print(k, "worst err/tol %.3f" % worst[k][0], worst[k][1], flag)


if __name__ == "__main__":
    main()
