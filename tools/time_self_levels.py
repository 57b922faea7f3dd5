"""Device time of the self levels vs the Gram at general order (development)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import _self_levels_t, gram_block  # noqa: E402

for n, L, d, M, p in ((1024, 128, 8, 5, 5), (1024, 128, 8, 5, 2), (4096, 64, 4, 4, 2)):
    cfg = KernelConfig(n_levels=M, order=p, normalization="levelwise")
    X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
    Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
    for _ in range(2):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        dx = _self_levels_t(X, cfg, "fp32")
        dy = _self_levels_t(Y, cfg, "fp32")
        e[1].record()
        gram_block(X, Y, cfg, diag_x=dx, diag_y=dy)
        e[2].record()
        torch.cuda.synchronize()
    print(f"n={n} L={L} d={d} M={M} p={p}: self levels {e[0].elapsed_time(e[1]):.1f} ms, "
          f"Gram {e[1].elapsed_time(e[2]):.1f} ms", flush=True)
