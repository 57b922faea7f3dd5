"""Which certification rule flags which entries at a config's shapes (development)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import sigkern_oracle as O  # noqa: E402
from paper_2501_07145_b200 import SeedStream, _native, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import gram_block  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
N, L, d, M, p, kind, norm, sym, _ = bench.CONFIGS[name]
cfg = bench.kernel_config(name)
X = torch.from_numpy(gen_brownian(n, L, d, SeedStream(1)).data).cuda()
Y = torch.from_numpy(gen_brownian(n, L, d, SeedStream(2)).data).cuda()
K0, lv = gram_block(X, Y, cfg, want_levels=True, flags=_native.SK_FLAG_NO_FIXUP)
K0, lv = K0.cpu().numpy(), lv.cpu().numpy()
Xh, Yh = X.cpu().numpy(), Y.cpu().numpy()
G = O.point_gram(O.static_params(kind), Xh[:, None, [0, -1]], Yh[None, :, [0, -1]])
k1 = G[..., 1, 1] - G[..., 0, 1] - G[..., 1, 0] + G[..., 0, 0]
S = np.abs(lv).sum(-1)
tau = 0.15 if kind == "linear" else 0.01
f_tau = np.abs(K0) < tau * S
f_noise = np.abs(lv[..., 1] - k1) > 1e-4 * np.abs(K0)
print(name, "n", n, "tau-rule", int(f_tau.sum()), "noise-rule", int(f_noise.sum()), "of", K0.size)
rows_hit = np.bincount(np.nonzero(f_tau | f_noise)[0], minlength=K0.shape[0])
print("flagged per row: max", rows_hit.max(), "mean", rows_hit.mean(), "rows with any", int((rows_hit > 0).sum()))
for a, b in zip(*np.nonzero(f_tau | f_noise)):
    print("  entry", a, b, "K %.4e" % K0[a, b], "levels", np.array2string(lv[a, b], precision=3),
          "k1 exact %.6e dev %.2e" % (k1[a, b], abs(lv[a, b, 1] - k1[a, b])))
    if a > 5:
        break
