"""Golden files for the dual bench cells and the analytic counters, produced by
the REFERENCE (benchmarks.py:170-234, utils.py:10-40, kernels.py:530-600).

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_bench_golden.py

Writes tests/golden/bench/<case>.cfg + <case>.out.csv (the reference CLI's
`bench` CSV with wall_time = false, so every byte is deterministic) and
tests/golden/counts.json (ResourceCounters flops / peak_bytes of
sig_kernel_gram calls over shapes, normalisations, tilings and algorithms).
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sigkern.cli import main  # noqa: E402
from sigkern.kernels import KernelConfig, sig_kernel_gram  # noqa: E402
from sigkern.rng import SeedStream  # noqa: E402
from sigkern.sequences import gen_brownian  # noqa: E402
from sigkern.static.kernels import StaticKernelSpec  # noqa: E402
from sigkern.utils import ResourceCounters  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
BENCH = os.path.join(HERE, "bench")

CASES = {
    "dual_fixed_bw": ["bench.methods = dual_dp, dual_pde", "bench.n_list = 6, 9",
                      "bench.l_list = 12, 20", "bench.m_list = 2, 4", "bench.dim = 3",
                      "kernel.static.bandwidth = 1.5", "bench.wall_time = false"],
    "dual_median_order": ["bench.methods = dual_dp", "bench.n_list = 8", "bench.l_list = 30",
                          "bench.m_list = 0, 3, 5", "bench.order = none", "bench.dim = 2",
                          "bench.wall_time = false", "seed = 11"],
    "dual_linear_nodiff": ["bench.methods = dual_dp, dual_pde", "bench.n_list = 5",
                           "bench.l_list = 9", "bench.m_list = 3", "bench.difference = false",
                           "kernel.static.kind = linear", "kernel.static.bandwidth = 2.0",
                           "bench.wall_time = false"],
}

COUNT_CASES = [
    # (nx, lx, ny or None, ly, d, M, order, difference, normalization, algorithm, tile_memory)
    (7, 10, 5, 8, 2, 3, 1, True, "none", "dp", 256 * 2 ** 20),
    (7, 10, None, 10, 2, 4, 2, True, "levelwise", "dp", 256 * 2 ** 20),
    (9, 12, None, 12, 3, 5, 5, True, "global", "dp", 20000),      # several tiles, symmetric
    (9, 12, 6, 7, 3, 3, 1, True, "levelwise", "dp", 30000),        # several tiles, cross
    (4, 6, 3, 6, 2, 0, 1, True, "none", "dp", 256 * 2 ** 20),      # M = 0
    (4, 1, 3, 6, 2, 3, 1, True, "none", "dp", 256 * 2 ** 20),      # one-point sequences
    (5, 7, 4, 9, 2, 3, 2, False, "levelwise", "dp", 256 * 2 ** 20),
    (6, 10, 4, 12, 2, 3, 1, True, "none", "pde", 256 * 2 ** 20),
    (6, 10, None, 10, 2, 3, 1, True, "global", "pde", 5000),
    (5, 8, 3, 6, 3, 3, 1, False, "global", "pde", 256 * 2 ** 20),
    (1, 1000, None, 1000, 2, 2, 1, True, "none", "dp", 256 * 2 ** 20),  # criterion 09 shapes
    (1, 2000, None, 2000, 2, 2, 1, True, "none", "dp", 256 * 2 ** 20),
]


def make_bench():
    os.makedirs(BENCH, exist_ok=True)
    for name, lines in CASES.items():
        cfg = os.path.join(BENCH, f"{name}.cfg")
        with open(cfg, "w") as fh:
            fh.write("\n".join(["command = bench"] + lines) + "\n")
        out = os.path.join(BENCH, f"{name}.out.csv")
        rc = main(["bench", "--config", cfg, "--output", out])
        assert rc == 0, (name, rc)


def make_counts():
    rows = []
    for k, (nx, lx, ny, ly, d, M, order, diff, norm, algo, tm) in enumerate(COUNT_CASES):
        X = gen_brownian(nx, lx, d, SeedStream(100 + k)).data if lx >= 2 else \
            np.zeros((nx, lx, d)) + np.arange(nx)[:, None, None] * 0.1
        Y = None if ny is None else gen_brownian(ny, ly, d, SeedStream(200 + k)).data
        cfg = KernelConfig(static=StaticKernelSpec(kind="rbf", bandwidth=1.3), n_levels=M,
                           order=order, difference=diff, normalization=norm)
        c = ResourceCounters()
        sig_kernel_gram(X, Y, cfg=cfg, algorithm=algo, counters=c, tile_memory=tm)
        rows.append({"nx": nx, "lx": lx, "ny": ny, "ly": ly, "d": d, "M": M, "order": order,
                     "difference": diff, "normalization": norm, "algorithm": algo,
                     "tile_memory": tm, "flops": c.flops, "peak_bytes": c.peak_bytes})
    with open(os.path.join(HERE, "counts.json"), "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    make_bench()
    make_counts()
