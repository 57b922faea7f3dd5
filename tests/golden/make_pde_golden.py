"""Golden vectors for the PDE path (algorithm="pde", kernels.py:334-507), produced by
the REFERENCE itself. Run in the build container:

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_pde_golden.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sigkern import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian, sig_kernel_gram  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    out = {}
    cases = [
        ("rbf_cross", "rbf", dict(bandwidth=1.3), True, "none", False, (5, 9, 3), (4, 7, 3)),
        ("rbf_sym_global", "rbf", dict(bandwidth=0.8), True, "global", True, (6, 8, 2), None),
        ("linear_cross", "linear", dict(scale=0.7), True, "none", False, (4, 10, 2), (3, 6, 2)),
        ("matern32_cross", "matern32", dict(bandwidth=1.1), True, "none", False, (3, 6, 2), (4, 5, 2)),
        ("rbf_nodiff", "rbf", dict(bandwidth=1.0), False, "none", False, (3, 4, 2), (2, 5, 2)),
        ("rbf_long", "rbf", dict(bandwidth=1.0), True, "global", False, (3, 64, 4), (2, 50, 4)),
    ]
    for name, kind, st, diff, norm, sym, xs, ys in cases:
        X = gen_brownian(*xs, SeedStream(11, (name,))).data
        Y = None if sym else gen_brownian(*ys, SeedStream(12, (name,))).data
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **st), difference=diff,
                           normalization=norm)
        K = sig_kernel_gram(X, Y, cfg=cfg, algorithm="pde")
        out[f"{name}__X"] = X
        if Y is not None:
            out[f"{name}__Y"] = Y
        out[f"{name}__K"] = K
        out[f"{name}__kind"] = np.array(kind)
        out[f"{name}__param"] = np.array(list(st.values())[0])
        out[f"{name}__diff"] = np.array(diff)
        out[f"{name}__norm"] = np.array(norm)
    np.savez_compressed(os.path.join(HERE, "pde.npz"), **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
