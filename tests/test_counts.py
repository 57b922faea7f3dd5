"""ResourceCounters of sig_kernel_gram follow the reference's analytic model
term for term (utils.gram_counts vs reference counters captured by
tests/golden/make_bench_golden.py), incl. the dual-DP peak-bytes scaling the
reference's acceptance criterion 09 checks (test_acceptance.py:266-300)."""

import json
import os

import pytest

from paper_2501_07145_b200.utils import ResourceCounters, gram_counts

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "counts.json")
ROWS = json.load(open(GOLDEN))


@pytest.mark.parametrize("row", ROWS, ids=[f"{r['algorithm']}-{k}" for k, r in enumerate(ROWS)])
def test_gram_counts_match_reference(row):
    c = ResourceCounters()
    sym = row["ny"] is None
    gram_counts(c, row["nx"], row["lx"], row["nx"] if sym else row["ny"],
                row["lx"] if sym else row["ly"], row["d"], row["M"],
                max(1, min(row["order"], row["M"])) if row["M"] >= 1 else 1,
                row["difference"], row["normalization"], sym, row["algorithm"],
                row["tile_memory"])
    assert (c.flops, c.peak_bytes) == (row["flops"], row["peak_bytes"])


def test_criterion_09_dual_dp_bytes_quadratic_in_L():
    peaks = {r["lx"]: r["peak_bytes"] for r in ROWS if r["nx"] == 1 and r["algorithm"] == "dp"}
    assert 3.5 <= peaks[2000] / peaks[1000] <= 4.5
    mine = {}
    for L in (1000, 2000):
        c = ResourceCounters()
        gram_counts(c, 1, L, 1, L, 2, 2, 1, True, "none", True)
        mine[L] = c.peak_bytes
    assert mine == peaks
