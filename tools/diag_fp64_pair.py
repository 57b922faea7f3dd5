"""Time of the float64 kernel for a few pairs at a config's shapes (development)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_07145_b200 import SeedStream, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import gram_block  # noqa: E402

name = sys.argv[1]
N, L, d, M, p, kind, norm, sym, _ = bench.CONFIGS[name]
cfg = bench.kernel_config(name)
for n in (1, 4, 32):
    X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
    Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
    gram_block(X, Y, cfg, precision="fp64")
    torch.cuda.synchronize()
    t = time.perf_counter()
    gram_block(X, Y, cfg, precision="fp64")
    torch.cuda.synchronize()
    print(name, "fp64 pairs", n * n, "ms %.2f" % ((time.perf_counter() - t) * 1e3), flush=True)
