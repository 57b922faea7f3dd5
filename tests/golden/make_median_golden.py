"""Golden vectors for median_heuristic, produced by the REFERENCE itself
(static/kernels.py:165-187). Run in the build container:

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_median_golden.py
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sigkern import SeedStream, gen_brownian  # noqa: E402
from sigkern.static.kernels import median_heuristic  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(7)
    cases = {
        "pooled": (gen_brownian(8, 50, 3, SeedStream(1)).data.reshape(-1, 3), 1_000_000),
        "subsampled": (rng.standard_normal((2000, 4)), 1_000_000),  # 2M pairs > budget
        "tight_budget": (rng.standard_normal((60, 5)), 100),
        "three": (np.array([[0.0, 0.0], [3.0, 4.0], [6.0, 8.0]]), 1_000_000),
        "c3_points": (gen_brownian(4, 256, 16, SeedStream(1)).data.reshape(-1, 16), 1_000_000),
    }
    out = {}
    for name, (X, mp) in cases.items():
        out[f"{name}__X"] = X
        out[f"{name}__max_pairs"] = np.array(mp)
        out[f"{name}__median"] = np.array(median_heuristic(X, max_pairs=mp))
    np.savez_compressed(os.path.join(HERE, "median.npz"), **out)
    print({k: float(v) for k, v in out.items() if k.endswith("__median")})


if __name__ == "__main__":
    main()
