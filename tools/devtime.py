"""Device timing of one config's Gram at a chosen N (development helper, not a bench line).

    python tools/devtime.py c2 256 [fp32|fp64] [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2501_07145_b200.kernels import _self_levels_t, gram_block  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
# 5th argument "nofix": SK_FLAG_NO_FIXUP (time the FP32 kernels without the certification pass)
from paper_2501_07145_b200 import _native  # noqa: E402
flags = _native.SK_FLAG_NO_FIXUP if len(sys.argv) > 5 and sys.argv[5] == "nofix" else 0
# ad-hoc shapes: name "L<len>d<dim>M<levels>", e.g. L256d4M8 (rbf, order 1, unnormalised)
if name not in bench.CONFIGS:
    import re
    L_, d_, M_ = (int(v) for v in re.match(r"L(\d+)d(\d+)M(\d+)", name).groups())
    bench.CONFIGS[name] = (n, L_, d_, M_, 1, "rbf", "none", False, 2)
N, L, d, M, p, kind, norm, sym, _ = bench.CONFIGS[name]
cfg = bench.kernel_config(name)
rng = np.random.default_rng(0)
X = torch.from_numpy(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L - 1), axis=1)).cuda()
Y = torch.from_numpy(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L - 1), axis=1)).cuda()
F = bench.flops_per_entry(L, d, M)
peak = torch.cuda.get_device_properties(0).multi_processor_count * 128 * 2 * 1.965e-3
for it in range(reps):
    dx = dy = None
    if norm != "none":
        dx = _self_levels_t(X, cfg, prec, flags=flags)
        dy = _self_levels_t(Y, cfg, prec, flags=flags)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    K, _ = gram_block(X, Y, cfg, precision=prec, diag_x=dx, diag_y=dy, flags=flags)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tf = n * n * F / ms / 1e9
    print(f"{name} n={n} prec={prec} gram_ms={ms:.2f} entries/s={n*n/ms*1e3:.3e} "
          f"TFLOP/s={tf:.2f} frac={tf/peak:.3f} nan={int(torch.isnan(K).sum())}", flush=True)
