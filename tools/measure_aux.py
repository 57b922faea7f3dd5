"""Device timing of the paths around the Gram (§8(f) rows), next to the CPU oracle.

    python tools/measure_aux.py [out.json]

* PDE kernel (algorithm="pde", float64): K(X, Y), N = M' = 256, L = 64, d = 4.
* rfsf_exact_gram (float64 lifted DP): rfsf_full rff map, D = 16, n_levels 4,
  N = M' = 512, L = 32, d = 3.
* median_heuristic: 8192 points, d = 16.
Each device number is the median of 5 CUDA-event timed calls after a warm-up,
inputs resident on the device; the CPU number times the oracle on a bounded
sample (stated) with all host threads where the oracle uses them.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import sigkern_oracle as O  # noqa: E402
from paper_2501_07145_b200 import (KernelConfig, SeedStream, StaticKernelSpec, gen_brownian,  # noqa: E402
                                   median_heuristic, sig_kernel_gram)
from paper_2501_07145_b200.features import (SigFeatureConfig, StaticFeatureSpec,  # noqa: E402
                                            fit_sig_features, rfsf_exact_gram)


def dev_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


def cpu_s(fn):
    t = time.perf_counter()
    fn()
    return time.perf_counter() - t


res = {}
# PDE
X = gen_brownian(256, 64, 4, SeedStream(1)).data
Y = gen_brownian(256, 64, 4, SeedStream(2)).data
Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
cfg = KernelConfig(static=StaticKernelSpec(kind="rbf"), normalization="none")
ms = dev_ms(lambda: sig_kernel_gram(Xt, Yt, cfg=cfg, algorithm="pde"))
k = 8
cs = cpu_s(lambda: O.pde_gram(X[:k], Y[:k], sp=O.static_params("rbf")))
res["pde"] = {"workload": "algorithm='pde' K(X,Y) N=M'=256 L=64 d=4 rbf, float64",
              "device_ms": ms, "entries_per_s": 256 * 256 / (ms / 1e3),
              "cpu_oracle_entries_per_s": k * k / cs, "cpu_sample": f"{k}x{k} entries, 1 thread"}
# rfsf_exact_gram
Xr = gen_brownian(512, 32, 3, SeedStream(3)).data
Yr = gen_brownian(512, 32, 3, SeedStream(4)).data
fc = SigFeatureConfig(variant="rfsf_full", static=StaticFeatureSpec(kind="rff"), n_components=16,
                      projection=16, n_levels=4, order=1)
st = fit_sig_features(fc, Xr, SeedStream(5))
Xrt, Yrt = torch.from_numpy(Xr).cuda(), torch.from_numpy(Yr).cuda()
ms = dev_ms(lambda: rfsf_exact_gram(st, Xrt, Yrt, normalize=True))
k = 16
slots = [dict(kind="rff", n_components=16, weights=s.weights) for s in st.slot_states]
cs = cpu_s(lambda: O.rfsf_exact_gram(slots, Xr[:k], Yr[:k], M=4, p=1, normalize=True))
res["rfsf_exact_gram"] = {
    "workload": "rfsf_full rff D=16 (32 features/slot) n_levels=4 normalize N=M'=512 L=32 d=3, float64",
    "device_ms": ms, "entries_per_s": 512 * 512 / (ms / 1e3),
    "cpu_oracle_entries_per_s": k * k / cs, "cpu_sample": f"{k}x{k} entries (numpy BLAS)"}
# median heuristic
P = np.random.default_rng(0).standard_normal((8192, 16))
Pt = torch.from_numpy(P).cuda()
ms = dev_ms(lambda: median_heuristic(Pt))
cs = cpu_s(lambda: O.median_heuristic(P[:2048]))
res["median_heuristic"] = {"workload": "median_heuristic 8192 points d=16 (33.5M pairs, subsampled to <= 1e6)",
                           "device_ms": ms, "cpu_oracle_s_2048_points": cs}
res["gpu"] = torch.cuda.get_device_name(0)
out = sys.argv[1] if len(sys.argv) > 1 else None
txt = json.dumps(res, indent=1)
print(txt)
if out:
    open(out, "w").write(txt + "\n")
