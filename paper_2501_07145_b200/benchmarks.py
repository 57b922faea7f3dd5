"""Scalability sweep of the dual methods on the B200 path (reference:
sigkern/benchmarks.py:83-234).

`run_bench` mirrors the reference's sweep for its dual cells — `dual_dp`
(`sig_kernel_gram(..., algorithm="dp")`, the north-star path) and `dual_pde`
(`algorithm="pde"`) — with the same data streams (`gen_brownian` on
`seed.child(f"data_n{N}_l{L}")`, :178-179), the same median bandwidth
(:180-183), and the same `BenchRecord` fields: `wall_ms` (host perf_counter
around the call, :209/:230; the call returns host numpy, so it includes the
device work and both copies), `flop_count` / `peak_bytes_est` from
`ResourceCounters` (the reference's analytic model, utils.gram_counts), F = N
for dual methods (:215). `write_bench_csv` writes the reference's CSV layout
(:107-125).

The primal random-feature methods (rfsf_full, dp, dp1d, trp, ts) are outside
the B200 dual path: requesting one raises NotImplementedError.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, fields

from .config import KernelConfig, StaticKernelSpec
from .kernels import sig_kernel_gram
from .sequences import SeedStream, gen_brownian
from .static_kernels import median_heuristic
from .utils import ResourceCounters
from .wire import format_value

__all__ = ["BenchRecord", "BenchSettings", "run_bench", "write_bench_csv", "bench_header",
           "DUAL_METHODS", "PRIMAL_METHODS", "BENCH_METHODS"]

DUAL_METHODS = ("dual_dp", "dual_pde")                      # benchmarks.py:44
PRIMAL_METHODS = ("rfsf_full", "dp", "dp1d", "trp", "ts")   # benchmarks.py:45
BENCH_METHODS = DUAL_METHODS + PRIMAL_METHODS


@dataclass
class BenchRecord:
    """One measured (method, problem size) cell (benchmarks.py:83-104)."""

    method: str
    N: int
    L: int
    d: int
    M: int
    p: int
    D: int
    Q: int
    F: int
    wall_ms: float
    flop_count: int
    peak_bytes_est: int
    mape: float | None = None


def bench_header() -> list:
    return [f.name for f in fields(BenchRecord)]


def write_bench_csv(path, records) -> None:
    """benchmarks.py:111-125: header line, empty cells for None."""
    lines = [",".join(bench_header())]
    for r in records:
        row = []
        for f in fields(BenchRecord):
            v = getattr(r, f.name)
            if v is None:
                row.append("")
            elif isinstance(v, str):
                row.append(v)
            else:
                row.append(format_value(v))
        lines.append(",".join(row))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


@dataclass(frozen=True)
class BenchSettings:
    """Sweep grid and switches (benchmarks.py:129-152; same fields, defaults, checks)."""

    methods: tuple = BENCH_METHODS
    n_list: tuple = (10,)
    l_list: tuple = (100,)
    dq_list: tuple = (100,)  # D = Q for every primal method
    m_list: tuple = (5,)
    dim: int = 5
    order: int | None = 1
    difference: bool = True
    static_kind: str = "rbf"
    bandwidth: float | str = "median"
    n_seeds: int = 1
    compute_mape: bool = False
    wall_time: bool = True

    def __post_init__(self):
        for m in self.methods:
            if m not in BENCH_METHODS:
                raise ValueError(f"unknown bench method {m!r}; choose from {BENCH_METHODS}")
        if self.n_seeds < 1:
            raise ValueError(f"n_seeds must be >= 1, got {self.n_seeds}")


def run_bench(settings: BenchSettings, seed: SeedStream, n_threads: int = 1, *,
              precision: str = "fp32") -> list:
    """Run the sweep; records in (N, L, DQ, M) x methods order (benchmarks.py:170-203)."""
    primal = [m for m in settings.methods if m not in DUAL_METHODS]
    if primal:
        raise NotImplementedError(
            f"bench methods {tuple(primal)} are primal random-feature methods, outside the "
            f"B200 dual path; supported: {DUAL_METHODS}")
    if not isinstance(seed, SeedStream):
        seed = SeedStream(int(seed))
    records = []
    for N in settings.n_list:
        for L in settings.l_list:
            data = gen_brownian(int(N), int(L), settings.dim, seed.child(f"data_n{N}_l{L}"))
            if settings.bandwidth == "median":
                bw = median_heuristic(data.data.reshape(-1, data.dim))
            else:
                bw = float(settings.bandwidth)
            for DQ in settings.dq_list:
                for M in settings.m_list:
                    p = settings.order if settings.order is not None else M
                    p = min(max(p, 1), max(M, 1))
                    kcfg = KernelConfig(
                        static=StaticKernelSpec(kind=settings.static_kind, bandwidth=bw),
                        n_levels=int(M), order=settings.order,
                        difference=settings.difference)
                    # compute_mape only feeds the primal cells' MAPE (benchmarks.py:192-197);
                    # dual records carry mape=None either way
                    for method in settings.methods:
                        records.append(_bench_cell(method, data, kcfg, settings, int(N), int(L),
                                                   int(DQ), int(M), p, n_threads, precision))
    return records


def _bench_cell(method, data, kcfg, settings, N, L, DQ, M, p, n_threads,
                precision) -> BenchRecord:
    # benchmarks.py:206-234, dual branch
    counters = ResourceCounters()
    t0 = time.perf_counter()
    algo = "dp" if method == "dual_dp" else "pde"
    sig_kernel_gram(data, cfg=kcfg, algorithm=algo, n_threads=n_threads, counters=counters,
                    precision=precision)
    wall = (time.perf_counter() - t0) * 1e3 if settings.wall_time else 0.0
    return BenchRecord(method=method, N=N, L=L, d=settings.dim, M=M, p=p, D=DQ, Q=DQ, F=N,
                       wall_ms=wall, flop_count=counters.flops,
                       peak_bytes_est=counters.peak_bytes, mape=None)
