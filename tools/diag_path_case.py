"""Details of one tools/path_sweep.py case: per-level FP32 vs float64 of the worst
entry and of its self levels (development; python tools/diag_path_case.py seed)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, _native, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import _self_levels_t, gram_block  # noqa: E402

KINDS = ("rbf", "linear", "matern12", "matern32", "matern52", "rational_quadratic")
seed = int(sys.argv[1])
r = np.random.default_rng(9000 + seed)
kind = KINDS[int(r.integers(0, len(KINDS)))]
M = int(r.integers(1, 9))
p = 1 if r.random() < 0.4 else int(r.integers(1, M + 1))
norm = ("none", "levelwise", "global")[int(r.integers(0, 3))]
diff = bool(r.random() < 0.8)
d = int((2, 3, 5, 8, 13, 16, 20, 40)[int(r.integers(0, 8))])
lx, ly = int(r.integers(2, 120)), int(r.integers(2, 120))
if r.random() < 0.3:
    lx, ly = int(r.integers(6, 30)), int(r.integers(6, 30))
kw = {}
if kind != "linear":
    kw["bandwidth"] = float(r.uniform(0.4, 2.0))
else:
    kw["scale"] = float(r.uniform(0.3, 1.5))
if kind == "rational_quadratic":
    kw["alpha"] = float(r.uniform(0.5, 3.0))
print(kind, kw, "M", M, "p", p, norm, "diff", diff, "d", d, "L", lx, ly)
X = torch.from_numpy(gen_brownian(6, lx, d, SeedStream(seed, ("x",))).data).cuda()
Y = torch.from_numpy(gen_brownian(5, ly, d, SeedStream(seed, ("y",))).data).cuda()
mk = lambda nm: KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=p,
                             difference=diff, normalization=nm)
K = gram_block(X, Y, mk(norm))[0].cpu().numpy()
K6 = gram_block(X, Y, mk(norm), precision="fp64")[0].cpu().numpy()
e = np.abs(K - K6) / np.abs(K6)
i, j = np.unravel_index(np.argmax(e), e.shape)
print("worst", (i, j), "err %.2e" % e[i, j], "K %.6e" % K6[i, j])
K0, lv0 = gram_block(X, Y, mk("none"), want_levels=True, flags=_native.SK_FLAG_NO_FIXUP)
_, lv6 = gram_block(X, Y, mk("none"), want_levels=True, precision="fp64")
for m in range(M + 1):
    a, b = lv0[i, j, m].item(), lv6[i, j, m].item()
    print(f" level {m}: f64 {b: .6e} fp32 {a: .6e} rel {abs(a - b) / max(abs(b), 1e-300):.2e}")
for nm, Z, k in (("x", X, i), ("y", Y, j)):
    s32 = _self_levels_t(Z, mk("none"), "fp32", flags=_native.SK_FLAG_NO_FIXUP)[k].cpu().numpy()
    s32c = _self_levels_t(Z, mk("none"), "fp32")[k].cpu().numpy()
    s64 = _self_levels_t(Z, mk("none"), "fp64")[k].cpu().numpy()
    print(f" self {nm}: rel raw {np.array2string(np.abs(s32 - s64) / np.abs(s64), precision=2)}"
          f" certified {np.array2string(np.abs(s32c - s64) / np.abs(s64), precision=2)}")
