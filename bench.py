"""Benchmark: signature-kernel Gram entries/s and % of the FP32 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

Default workload (BASELINE.json configs[2], the metric's headline config):
normalised (levelwise) order-1 RBF signature kernel, n_levels=5, cross Gram
K(X, Y) of N = M' = 8192 random-walk sequences, L = 256, d = 16, float64
inputs generated with the reference's own generator (restated bit for bit).

A "step" is one whole Gram: self levels of X and Y (normalisation) and the
fused Gram kernel with its normalisation epilogue. With N GPUs (torchrun) the
SAME Gram is sharded (strong scaling, the north star's "8192^2 Gram sharded
over 1/2/4/8 B200"): `distributed.sharded_gram` gives every rank a block of
rows, and the step includes each rank's self levels, its rows and the NCCL
all-gather that assembles K on every rank; it is timed as the max over ranks.
`value` is entries/s with inputs resident in HBM; `e2e` is the same through
the public API (`SignatureKernel.__call__`, or `sharded_gram` on N GPUs) from
pinned host float64 inputs to the host float64 Gram.
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # the CPU baseline mirrors BASELINE.md

import argparse
import json
import subprocess
import threading
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "signature-kernel entries/sec and % FP32 roofline at L=256,d=16,m=5 (1/2/4/8 GPU)"

# name: (N, L, d, n_levels, order, kind, normalization, symmetric, cpu sample k)
CONFIGS = {
    "c1": (64, 50, 3, 5, 1, "rbf", "levelwise", True, 64),
    "c2": (1024, 128, 8, 5, 5, "rbf", "none", False, 12),
    "c3": (8192, 256, 16, 5, 1, "rbf", "levelwise", False, 24),
    "c4": (4096, 128, 128, 3, 1, "linear", "none", False, 16),
    "c5": (512, 2048, 4, 8, 1, "rbf", "none", False, 2),
}


# measured FP32 pipe rate per SM per clock (FFMA2 / FADD2 at 8 warps/SM on the
# B200, tools/microbench/fp32_pipes.cu -> profiles/r2_fp32_pipes.txt; nominal 128)
FP32_LANE_OPS = 127.85


def flops_per_entry(L, d, M):
    """North-star algorithmic work per Gram entry: 2 L L' (d + 2M)."""
    return 2 * L * L * (d + 2 * M)


def order_aware_flops_per_entry(L, d, M, p):
    """Work the recursion actually does per entry at order p (SURVEY.md §8(d) note):
    2d per cell for the static stage, and per level m the min(m,p)^2 states with
    their row/column/total sums (about 2 flops per state: one multiply, one
    accumulate) plus 4 per level for the scans. Equals the north-star model at p = 1."""
    per_cell = 2 * d + sum(2 * min(m, p) ** 2 + 2 for m in range(1, M + 1)) if p > 1 else 2 * d + 4 * M
    return L * L * per_cell


def geo_ops_per_cell(M, p):
    """FP32 pipe slots per cell of the general-order recursion (p > 1): every
    FMUL / FADD / FFMA of the generated straight-line cell (sk_geo_cells.cuh,
    one slot each whether it is worth 1 or 2 flops), counted from the header
    the kernel compiles. The order-aware flop model above credits 2 flops per
    state and misses the weighted row, column and total sums the recursion
    needs (kernels.py:179-199), about 3 p^2 slots per level."""
    import re
    src = open(os.path.join(ROOT, "paper_2501_07145_b200", "csrc", "sk_geo_cells.cuh")).read()
    i = src.index(f"struct GeoCell<{M}, {p}>")
    body = src[i:src.index("};", i)]
    n = 0
    for ln in body.splitlines():
        ln = ln.strip()
        if "fmaf(" in ln or re.search(r"\+= ", ln) or re.search(r"= av \* ", ln):
            n += 1
    return n


def pipe_slot_frac(L, d, M, p, pairs, ms, sms, clk_mhz):
    """Share of the FP32 pipe's slots (148 SMs x 127.85 / clk) the p > 1 kernel
    fills with necessary work: the generated cell's ops plus the point stage's
    ~d + 6 (d FMAs of the inner product, the n-terms, the exp prescale and the
    double difference)."""
    slots = pairs * (L - 1) ** 2 * (geo_ops_per_cell(M, p) + d + 6)
    return slots / (ms / 1e3) / (sms * FP32_LANE_OPS * clk_mhz * 1e6)


def tensor_roofline(nx, ny, L, d, kind, call_ms):
    """3xTF32 cell-value GEMM work of one sk_gram call against the TF32 tensor peak
    (half the MEASURED_PEAKS.json dense bf16 burst figure; B200_PROFILING's
    2.25 PF/2 nominal if that file is absent). Timed over the whole call (GEMM + DP)."""
    rows = 2 * ((L + 1) // 2)
    K = ((d if kind == "linear" else d + 2) + 3) // 4 * 4  # rbf folds two n-terms (sk_gemm.cu)
    flops = 3 * 2 * (nx * rows) * (ny * rows) * K
    peak, src = 1125.0, "nominal 2.25 PF dense bf16 / 2 (B200_PROFILING.md fallback)"
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        try:
            peak = json.load(open(mp))["bf16_tflops"] / 2
            src = "MEASURED_PEAKS.json bf16_tflops (burst) / 2"
        except (KeyError, ValueError):
            pass
    achieved = flops / (call_ms / 1e3) / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s (TF32)",
            "frac": achieved / peak, "flops_per_call": flops, "peak_source": src,
            "note": "3 MMAs (hi*hi, hi*lo, lo*hi) per k-step; time includes the DP kernel"}


def path_info(name):
    """(execution path, kernel label, own kernel launches per sk_gram / sk_self_levels call)."""
    from paper_2501_07145_b200.kernels import execution_path
    N, L, d, M, p, kind, norm, sym, _ = CONFIGS[name]
    path = execution_path(L, L, d, kernel_config(name))
    D = 4 if d <= 4 else (8 if d <= 8 else 16)
    # translation-invariant kinds: one midrange (centring) launch per input batch
    mr_gram = 0 if kind == "linear" else (1 if sym else 2)
    mr_self = 0 if kind == "linear" else 1
    if path == "fused":
        state = (f"LaneState1<PointStage<{D},8>,{M}>" if p == 1
                 else f"LaneStateG<PointStage<{D},4>,{M},{p}>")
        return path, f"sk::fast::gram_kernel<{state}> (fused Gram)", 3 + mr_gram, 3 + mr_self
    if path == "gemm":
        # x blocks of the 2 GiB cell-matrix budget (sk_gemm.cu block_rows); one DP launch each
        C = 8 if p == 1 else 4
        sw = 32 if L > 32 * C else 1 << max(0, (-(-L // C) - 1).bit_length())
        cols = sw * C * max(1, -(-L // (32 * C)))
        rows = 2 * ((L + 1) // 2)
        bx = max(1, min(N, (2 << 30) // (rows * N * cols * 4)))
        # per x block one tcgen05 GEMM launch and one DP launch, plus the two operand packs
        # (profiles/r1_c4_launches.txt: 32 + 32 + 2 per Gram at N = 1024)
        return (path, "sk::tc::tc_gemm_kernel (2-SM tcgen05 3xTF32 cell values) + "
                      "sk::gemm::gemm_dp_kernel (systolic DP); timed: the whole sk_gram call",
                2 + 2 * -(-N // bx) + mr_gram, 3 + mr_self)
    return path, "sk::generic_levels_kernel (float64)", 2, 2


def make_inputs(name, start=0):
    """X = sequences [start, start+N) of the SeedStream(1) batch, Y = the first N of SeedStream(2)."""
    from paper_2501_07145_b200 import SeedStream, gen_brownian
    N, L, d = CONFIGS[name][:3]
    X = gen_brownian(N, L, d, SeedStream(1), start=start).data
    Y = None if CONFIGS[name][7] else gen_brownian(N, L, d, SeedStream(2)).data
    return X, Y


def kernel_config(name):
    from paper_2501_07145_b200 import KernelConfig, StaticKernelSpec
    N, L, d, M, p, kind, norm, sym, _ = CONFIGS[name]
    return KernelConfig(static=StaticKernelSpec(kind=kind), n_levels=M, order=p,
                        normalization=norm)


def workload(name):
    N, L, d, M, p, kind, norm, sym, _ = CONFIGS[name]
    return {"workload": f"{name}: SignatureKernel n_levels={M} order={p} {kind} "
                        f"normalization={norm} {'K(X)' if sym else 'K(X,Y)'} N=M'={N} L={L} d={d}",
            "N": N, "L": L, "d": d, "n_levels": M, "order": p, "static": f"{kind}(1.0)",
            "normalization": norm, "symmetric": sym,
            "l2": "no flush: packed inputs + float64 Gram exceed the 126 MB L2" if N >= 4096
            else "small config (fits L2)"}


# ---------------------------------------------------------------------------
# CPU baseline (oracle port of the reference's algorithm; test infrastructure)
# ---------------------------------------------------------------------------

def cpu_sample(name, k=None, threads=None):
    from oracle import sigkern_oracle as O
    N, L, d, M, p, kind, norm, sym, kdef = CONFIGS[name]
    k = k or kdef
    threads = threads or O.host_threads()
    X = O.gen_brownian(k, L, d, 1)
    Y = None if sym else O.gen_brownian(k, L, d, 2)
    sp = O.static_params(kind)
    t0 = time.perf_counter()
    O.gram(X, Y, sp=sp, M=M, p=p, normalization=norm, n_threads=threads)
    dt = time.perf_counter() - t0
    return k * k / dt, dt, k, threads


def cpu_baseline_block(name):
    rate, dt, k, threads = cpu_sample(name)
    return {"value": rate, "unit": "entries/s", "cores": threads, "kind": "port",
            "sample": f"{name} {k}x{k} sub-block ({k*k} entries) via oracle/sigkern_oracle.py "
                      f"(numpy port of kernels.py:530-600), {dt:.2f} s, "
                      f"OPENBLAS_NUM_THREADS=1, n_threads={threads}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    name = args.config
    for _ in range(args.warmup):
        cpu_sample(name)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt, k, threads = cpu_sample(name)
        rates.append(r)
        times.append(dt)
    value = float(np.median(rates))
    line = {"metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(times)),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: gen_brownian random walks (SeedStream 1 / 2)",
            "config": workload(name), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "entries/s", "cores": threads, "kind": "port",
                             "sample": f"{name} {k}x{k} sub-block per step, oracle port of the "
                                       f"reference's numpy DP, n_threads={threads}"},
            "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: NVML polled
    every 10 ms from a thread (the data nvidia-smi reports), plus
    `sample_now()` from the main thread while the GPU is still busy, so even a
    sub-millisecond region (c1) gets samples. Falls back to `nvidia-smi -lms`."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nv = None
        self.lines = []

    def _nvml_line(self):
        nv, h = self.nv, self.handle
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        flags = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        act = ["Active" if r & f else "Not Active" for f in flags]
        return f"{sm}, {mx}, {r:#x}, " + ", ".join(act)

    def sample_now(self):
        if self.nv is not None:
            try:
                self.lines.append(self._nvml_line())
            except Exception:
                pass

    def _poll(self):
        while not self.stop.is_set():
            self.sample_now()
            self.stop.wait(0.01)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.handle = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.nv = nv
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.nv is not None:
            self.stop.set()
            self.thread.join(timeout=5)
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        load = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2501_07145_b200 import LinearKernel, RBFKernel, SignatureKernel
    from paper_2501_07145_b200.distributed import _default_compute, row_blocks, sharded_gram
    from paper_2501_07145_b200.kernels import _self_levels_t, gram_block

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo: test hook that runs the multi-rank logic on ONE GPU
    # (ranks share the device; collectives go through host tensors)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        tt = torch.tensor([v], device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    name = args.config
    N, L, d, M, p, kind, norm, sym, _ = CONFIGS[name]
    cfg = kernel_config(name)
    # Strong scaling (the north star's "8192^2 Gram sharded over 1/2/4/8 B200"):
    # every rank holds X and Y, evaluates its row block of the ONE fixed Gram
    # (distributed.sharded_gram: equal row blocks for K(X, Y), paired blocks
    # for K(X)) including the self levels of the normalisation, and one
    # all-gather over NVLink assembles K on every rank — all inside the step.
    Xh, Yh = make_inputs(name)
    X = torch.from_numpy(Xh).to(dev)
    Y = None if Yh is None else torch.from_numpy(Yh).to(dev)
    ny = N

    gram_ms = []  # CUDA events around this rank's Gram launches

    def timed_compute(Xa, Ya, cfga, r0, r1, precision, K_full=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        diag_x = diag_y = None
        if cfga.normalization != "none":  # self levels outside the Gram events
            diag_x = _self_levels_t(Xa, cfga, precision)
            diag_y = diag_x if Ya is None else _self_levels_t(Ya, cfga, precision)
        e0.record()
        K, _ = gram_block(Xa, Ya, cfga, row_begin=r0, row_end=r1, precision=precision,
                          diag_x=diag_x, diag_y=diag_y, K=K_full)
        e1.record()
        gram_ms.append((e0, e1))
        return K

    def step():
        if world == 1:
            return timed_compute(X, Y, cfg, 0, N, "fp32", None)
        return sharded_gram(X, Y, cfg, compute=timed_compute)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    gram_ms.clear()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        t0.record()
        for _ in range(args.steps):
            K = step()
        t1.record()
        clk.sample_now()  # the queued steps are still running
        barrier()
    elapsed = max_over_ranks(t0.elapsed_time(t1))
    ms = elapsed / args.steps
    entries = N * ny  # the one Gram, whatever the number of GPUs
    value = entries / (ms / 1e3)

    # dominant kernel: this rank's Gram launch(es), per step
    g_ms = float(np.sum([a.elapsed_time(b) for a, b in gram_ms])) / args.steps
    if world == 1:
        pairs = N * (N + 1) // 2 if sym else N * ny
    elif sym:
        from paper_2501_07145_b200.distributed import paired_row_blocks
        pairs = sum(sum(N - i for i in range(a, b)) for a, b in paired_row_blocks(N, world)[rank])
    else:
        r0, r1 = row_blocks(N, world)[rank]
        pairs = (r1 - r0) * ny
    F = flops_per_entry(L, d, M)
    achieved = pairs * F / (g_ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and world == 1:  # measured for the full-size single-GPU launch
        t = json.load(open(tpath)).get(name)
        if t:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    props = torch.cuda.get_device_properties(dev)
    clocks = clk.summary()
    sm_max = clocks["sm_max_mhz"] or 1965.0
    peak = props.multi_processor_count * FP32_LANE_OPS * 2 * sm_max * 1e6 / 1e12

    # end to end through the public API from pinned host buffers: the
    # SignatureKernel facade (1 GPU) or distributed.sharded_gram (N GPUs; every
    # rank copies X and Y in and the assembled K out)
    Xp = torch.from_numpy(Xh).pin_memory()
    Yp = None if Yh is None else torch.from_numpy(Yh).pin_memory()
    Kh = torch.empty((N, ny), dtype=torch.float64).pin_memory()
    static = RBFKernel(1.0) if kind == "rbf" else LinearKernel(1.0)
    sk = SignatureKernel(n_levels=M, order=p, normalization=norm, static_kernel=static)

    def e2e_step():
        Xd = Xp.to(dev, non_blocking=True)
        Yd = None if Yp is None else Yp.to(dev, non_blocking=True)
        Kd = sk(Xd, Yd) if world == 1 else sharded_gram(Xd, Yd, cfg)
        Kh.copy_(Kd, non_blocking=True)
        return Kd

    e2e_step()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.e2e_steps):
        e2e_step()
    b.record()
    barrier()
    e_ms = max_over_ranks(a.elapsed_time(b) / args.e2e_steps)
    h2d = Xh.nbytes + (0 if Yh is None else Yh.nbytes)
    e2e = {"value": entries / (e_ms / 1e3), "unit": "entries/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": N * ny * 8, "ms_per_step": e_ms,
           "api": ("SignatureKernel(...)(X, Y)" if world == 1 else
                   "distributed.sharded_gram(X, Y, cfg) on every rank") +
                  ", pinned host float64 in, host float64 K out (bytes per rank)"}

    path, klabel, per_gram, per_self = path_info(name)
    n_gram = 1 if world == 1 or not sym else 2  # symmetric: two row blocks per rank
    launches_per_step = n_gram * ((per_self if norm != "none" else 0) * (1 if sym else 2)
                                  + per_gram)
    if rank == 0:
        if world == 1:
            par = "single"
        elif sym:
            par = (f"paired row blocks x{world} (blocks r and {2 * world - 1}-r of {2 * world}), "
                   f"NCCL all_gather_into_tensor of the triangle rows + bitwise mirror")
        else:
            par = f"row blocks x{world} of the one {N}x{ny} Gram, NCCL all_gather_into_tensor"
        line = {
            "metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32 (float64 level sums and normalisation)",
            "data": "synthetic: gen_brownian random walks, SeedStream(1)/(2), reference "
                    "generator restated bit for bit",
            "config": dict(workload(name), parallelism=par),
            "e2e": e2e,
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_unit": "bytes per launch (ncu dram__bytes_read+write, profiles/traffic.json)",
                         "kernel": klabel + ", rank 0's sk_gram call(s) per step, CUDA events "
                                            "on its stream",
                         "path": path,
                         "flops_per_entry": F, "pairs_per_launch": pairs,
                         "order_aware_flops_per_entry": order_aware_flops_per_entry(L, d, M, p),
                         "order_aware_frac": (pairs * order_aware_flops_per_entry(L, d, M, p)
                                              / (g_ms / 1e3) / 1e12 / peak),
                         "kernel_ms": g_ms,
                         **({"pipe_slot_frac": pipe_slot_frac(L, d, M, p, pairs, g_ms,
                                                              props.multi_processor_count, sm_max),
                             "pipe_slot_note": "p > 1: FP32 instruction slots of the generated "
                                               "recursion cell + point stage, vs the pipe's "
                                               "slot rate (bench.py geo_ops_per_cell)"}
                            if 1 < p and path == "fused" else {}),
                         "peak_note": f"measured FP32 pipe rate: {props.multi_processor_count} "
                                      f"SMs x {FP32_LANE_OPS} lane-ops/clk (FFMA2/FADD2, "
                                      f"profiles/r2_fp32_pipes.txt) x 2 x {sm_max:.0f} MHz "
                                      f"(MEASURED_PEAKS.json has no FP32 figure)"},
            "cpu_baseline": cpu_baseline_block(name) if (world == 1 and not args.no_cpu) else None,
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
        }
        if path == "gemm":  # the tensor-core side, labelled (report both)
            line["roofline"]["tensor"] = tensor_roofline(N, ny, L, d, kind, g_ms)
        if world == 1:
            line["sample_check"] = sample_check(name, K, Xh, Yh)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def sample_check(name, K, Xh, Yh):
    """Max relative error of a few Gram entries against the float64 oracle."""
    from oracle import sigkern_oracle as O
    N, L, d, M, p, kind, norm, sym, _ = CONFIGS[name]
    idx = [(0, 0), (1, 5), (N - 1, N - 2), (N // 2, N // 3)]
    Kc = K.cpu().numpy() if hasattr(K, "cpu") else np.asarray(K)
    rows = sorted({i for i, _ in idx})
    cols = sorted({j for _, j in idx})
    Yref = Xh if Yh is None else Yh
    R = O.gram(Xh[rows], Yref[cols], sp=O.static_params(kind), M=M, p=p, normalization=norm)
    err = 0.0
    for i, j in idx:
        r = R[rows.index(i), cols.index(j)]
        err = max(err, abs(Kc[i, j] - r) / abs(r))
    return {"entries": idx, "max_rel_err": err}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--size", type=int, default=None,
                    help="override N (profiling runs only; not a bench line)")
    args = ap.parse_args()
    if args.size:
        c = list(CONFIGS[args.config])
        c[0] = args.size
        CONFIGS[args.config] = tuple(c)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
