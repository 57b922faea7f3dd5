"""Float64 order-1 Gram throughput (development)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import gram_block  # noqa: E402

for kind, n, L, d, M in (("rbf", 1024, 256, 16, 5), ("polynomial", 1024, 256, 16, 5),
                         ("rbf", 2048, 64, 4, 8), ("rbf", 512, 128, 1, 5)):
    kw = dict(degree=3, gamma=1.0) if kind == "polynomial" else {}
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, normalization="levelwise")
    X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
    Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
    gram_block(X[:8], Y[:8], cfg, precision="fp64")
    torch.cuda.synchronize()
    t = time.perf_counter()
    gram_block(X, Y, cfg, precision="fp64")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{kind} n={n} L={L} d={d} M={M}: fp64 {dt * 1e3:.1f} ms = {n * n / dt:.3g} entries/s", flush=True)
