"""Dump c4-shape FP32 level values next to float64 ones (development tool)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2501_07145_b200 import SeedStream, _native, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import gram_block  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
N, L, d, M, p, kind, norm, sym, _ = bench.CONFIGS[name]
cfg = bench.kernel_config(name)
X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
_, lv32 = gram_block(X, Y, cfg, flags=_native.SK_FLAG_NO_FIXUP, want_levels=True)
_, lv64 = gram_block(X, Y, cfg, precision="fp64", want_levels=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"dump_{name}.npz"), lv32=lv32.cpu().numpy(),
                    lv64=lv64.cpu().numpy())
print("dumped", lv32.shape)
