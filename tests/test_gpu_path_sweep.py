"""Every FP32 path against the float64 kernels on random configurations (the
generator of tools/path_sweep.py: kind, n_levels, order, normalisation,
difference, d 2-40, lengths 2-120 with a short-sequence bias), at the
north-star tolerances, plain relative error. The sweep that found the two
regimes now routed to float64; profiles/r2_path_sweep.txt has
~2,200 cases of it."""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import path_sweep  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("block", range(12))
def test_fp32_paths_within_tolerance(block):
    bad = []
    for seed in range(50000 + 60 * block, 50000 + 60 * (block + 1)):
        path, ratio, desc = path_sweep.run_case(seed)
        if path is not None and ratio > 1.0:
            bad.append((seed, path, round(ratio, 3), desc))
    assert not bad, bad
