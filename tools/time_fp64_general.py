"""Device time of float64 general-order Grams (development)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import execution_path, gram_block  # noqa: E402

for n, L, d, M, p, norm in ((256, 64, 2, 5, 3, "levelwise"), (256, 128, 8, 5, 5, "none"),
                            (1024, 128, 2, 4, 2, "none")):
    cfg = KernelConfig(n_levels=M, order=p, normalization=norm)
    X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
    gram_block(X[:8], X[:8], cfg, precision="fp64")
    torch.cuda.synchronize()
    t = time.perf_counter()
    gram_block(X, X, cfg, precision="fp64")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"n={n} L={L} d={d} M={M} p={p} {norm}: path(fp32)={execution_path(L, L, d, cfg)} "
          f"fp64 {dt * 1e3:.1f} ms = {n * n / dt:.3g} entries/s", flush=True)
