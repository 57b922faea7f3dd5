"""Far-end c3 golden block, produced by the REFERENCE: rows and columns
8168-8191 of the full-size c3 inputs (gen_brownian(8192, 256, 16) on
SeedStream(1) / SeedStream(2), sliced from the full batches), the 24 x 24
levelwise Gram (BASELINE.md §4's sub-block) and its unnormalised sum.

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_c3_far_golden.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sigkern import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian, sig_kernel_gram  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

if __name__ == "__main__":
    X = gen_brownian(8192, 256, 16, SeedStream(1)).data[8168:]
    Y = gen_brownian(8192, 256, 16, SeedStream(2)).data[8168:]
    out = {"X": X, "Y": Y, "rows": np.arange(8168, 8192)}
    for norm in ("levelwise", "none"):
        cfg = KernelConfig(static=StaticKernelSpec(kind="rbf", bandwidth=1.0), n_levels=5,
                           order=1, normalization=norm)
        out[f"K_{norm}"] = sig_kernel_gram(X, Y, cfg=cfg, n_threads=8)
    np.savez_compressed(os.path.join(HERE, "c3_far.npz"), **out)
