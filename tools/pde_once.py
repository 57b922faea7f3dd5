"""Two K(X, Y) calls of algorithm="pde" at the measure_aux shape (profiling helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import sig_kernel_gram  # noqa: E402

X = torch.from_numpy(gen_brownian(256, 64, 4, SeedStream(1)).data).cuda()
Y = torch.from_numpy(gen_brownian(256, 64, 4, SeedStream(2)).data).cuda()
for _ in range(2):
    sig_kernel_gram(X, Y, cfg=KernelConfig(), algorithm="pde")
torch.cuda.synchronize()
