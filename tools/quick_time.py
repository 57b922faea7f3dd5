"""Quick device timing of the c3 Gram at a given N (development helper)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2501_07145_b200 import KernelConfig, SeedStream, gen_brownian
from paper_2501_07145_b200.kernels import gram_block
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
L, d, M = 256, 16, 5
rng = np.random.default_rng(0)
X = torch.from_numpy(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L - 1), axis=1)).cuda()
Y = torch.from_numpy(np.cumsum(rng.standard_normal((n, L, d)) / np.sqrt(L - 1), axis=1)).cuda()
cfg = KernelConfig(n_levels=M, normalization="levelwise")
for it in range(3):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); K, _ = gram_block(X, Y, cfg); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    pairs = n * n + 2 * n
    F = 2 * L * L * (d + 2 * M)
    print(f"n={n} ms={ms:.1f} entries/s={n*n/ms*1e3:.3e} TFLOP/s={pairs*F/ms/1e9:.2f} frac74.4={pairs*F/ms/1e9/74.4:.3f}")
