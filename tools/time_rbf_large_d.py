"""rbf with d > 16 (float64 row-scan since round 2) vs linear on the GEMM-fed path (development)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import execution_path, gram_block  # noqa: E402

for kind, n, L, d in (("rbf", 512, 64, 24), ("rbf", 512, 64, 40), ("rbf", 256, 128, 24),
                      ("linear", 512, 64, 24)):
    cfg = KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=4, normalization="levelwise")
    X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
    gram_block(X[:4], X[:4], cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    gram_block(X, X, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{kind} n={n} L={L} d={d}: {execution_path(L, L, d, cfg)} {dt * 1e3:.1f} ms = {n * n / dt:.3g} entries/s",
          flush=True)
