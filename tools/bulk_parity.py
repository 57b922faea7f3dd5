"""Full-size parity sample (development / evidence tool): the FP32 Gram of a
BASELINE config at full size, and the float64 Gram of a random 64 x 64 subset
of its rows and columns (the float64 kernel, itself pinned to the reference at
1e-10); reports the relative-error distribution over those 4096 entries.

    python tools/bulk_parity.py <config> [rows] [seed]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2501_07145_b200 import SeedStream, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import sig_kernel_gram  # noqa: E402

name = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
N, L, d, M, p, kind, norm, sym, _ = bench.CONFIGS[name]
cfg = bench.kernel_config(name)
X = torch.from_numpy(gen_brownian(N, L, d, SeedStream(1)).data).cuda()
Y = torch.from_numpy(gen_brownian(N, L, d, SeedStream(2)).data).cuda()
K = sig_kernel_gram(X, Y, cfg=cfg)
rng = np.random.default_rng(seed)
ri = np.sort(rng.choice(N, k, replace=False))
ci = np.sort(rng.choice(N, k, replace=False))
R = sig_kernel_gram(X[ri], Y[ci], cfg=cfg, precision="fp64").cpu().numpy()
Kc = K[torch.from_numpy(ri).cuda()][:, torch.from_numpy(ci).cuda()].cpu().numpy()
err = np.abs(Kc - R) / np.abs(R)
tol = 1e-4 if norm == "none" else 1e-5
out = {"config": name, "entries": int(err.size), "max_rel_err": float(err.max()),
       "median_rel_err": float(np.median(err)), "p999_rel_err": float(np.percentile(err, 99.9)),
       "above_tol": int((err > tol).sum()), "tol": tol}
bad = np.argwhere(err > tol)
if len(bad):  # the worst offenders: their FP32 cancellation ratio |K| / sum_m |k_m|
    from paper_2501_07145_b200 import _native
    from paper_2501_07145_b200.kernels import gram_block
    Xs, Ys = X[torch.from_numpy(ri[bad[:4, 0]]).cuda()], Y[torch.from_numpy(ci[bad[:4, 1]]).cuda()]
    K0, lv = gram_block(Xs, Ys, cfg, want_levels=True, flags=_native.SK_FLAG_NO_FIXUP)
    lvc = lv.cpu().numpy()
    out["offenders"] = [{"err": float(err[a, b]), "K": float(R[a, b]),
                         "ratio": float(abs(lvc[q, q].sum()) / np.abs(lvc[q, q]).sum())}
                        for q, (a, b) in enumerate(bad[:4])]
print(json.dumps(out))
