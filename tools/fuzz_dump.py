"""Dump FP32 Gram / level values next to the float64 oracle for the seeded
random configurations of tests/test_gpu_fuzz.py (development tool for the
FP32 certification model; one npz per run).

    python tools/fuzz_dump.py <n_seeds> <out.npz>
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import sigkern_oracle as O  # noqa: E402
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian  # noqa: E402
from paper_2501_07145_b200.kernels import _self_levels_t, execution_path, gram_block  # noqa: E402
from test_gpu_fuzz import _case  # noqa: E402


def main():
    n, out = int(sys.argv[1]), sys.argv[2]
    res = {}
    for seed in range(n):
        kind, kw, M, order, norm, diff, d, lx, ly, sym = _case(seed)
        X = gen_brownian(5, lx, d, SeedStream(seed, ("x",))).data
        Y = X if sym else gen_brownian(4, ly, d, SeedStream(seed, ("y",))).data
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=order,
                           difference=diff, normalization="none")
        path = execution_path(lx, ly if not sym else lx, d, cfg)
        if path == "fp64":
            continue
        sp = O.static_params(kind, **kw)
        p = max(1, min(order, M))
        lvR = O.gram_levels(sp, X, Y, M, p, diff)
        dxR = O.self_levels(sp, X, M, p, diff)
        dyR = O.self_levels(sp, Y, M, p, diff)
        Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
        try:
            _, lv = gram_block(Xt, Yt, cfg, want_levels=True)
            dx = _self_levels_t(Xt, cfg, "fp32")
            dy = _self_levels_t(Yt, cfg, "fp32")
        except Exception as e:  # noqa: BLE001
            print(seed, "error", e)
            continue
        for k, v in (("lv", lv), ("dx", dx), ("dy", dy)):
            res[f"{seed}_{k}32"] = v.cpu().numpy()
        res[f"{seed}_lvR"], res[f"{seed}_dxR"], res[f"{seed}_dyR"] = lvR, dxR, dyR
        res[f"{seed}_meta"] = np.array([M, p, lx, ly, d, int(sym), int(diff)])
        res[f"{seed}_kind"] = np.array(kind)
        res[f"{seed}_norm"] = np.array(norm)
    np.savez_compressed(out, **res)
    print("dumped", len([k for k in res if k.endswith("_meta")]), "seeds")


if __name__ == "__main__":
    main()
