"""Calibration of the FP32 paths' per-level error (development tool; the
measurements behind the certification bound in csrc/sk_common.cuh).

For random configurations it records, per level m, the FP32 error of the
cross level values relative to the Cauchy-Schwarz scale of that level,
    a_m = max_pairs |k32_m(x,y) - k_m(x,y)| / sqrt(k_m(x,x) k_m(y,y)),
and of the self levels, s_m = max |k32_m(x,x) - k_m(x,x)| / k_m(x,x), with the
float64 oracle as truth. One JSON line per case.

    python tools/calib_fp32_error.py <n_cases> <seed> > out.jsonl
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sigkern_oracle as O  # noqa: E402
from paper_2501_07145_b200 import KernelConfig, StaticKernelSpec  # noqa: E402
from paper_2501_07145_b200.kernels import _self_levels_t, execution_path, gram_block  # noqa: E402

KINDS = ("rbf", "rbf", "rbf", "linear", "matern12", "matern32", "matern52", "rational_quadratic")


def case(r):
    kind = KINDS[int(r.integers(0, len(KINDS)))]
    order = 1 if r.random() < 0.7 else int(r.integers(2, 6))
    M = 8 if order == 1 else 5
    L = int(2 ** r.uniform(1.6, 11.0))
    ly = L if r.random() < 0.5 else int(2 ** r.uniform(1.6, 11.0))
    d = int((1, 2, 3, 4, 5, 8, 13, 16, 20, 33)[int(r.integers(0, 10))])
    bw = float(2 ** r.uniform(-1.5, 2.0))
    amp = float(10 ** r.uniform(-2.5, 1.0)) if r.random() < 0.3 else 1.0
    off = float(r.choice([0.0, 0.0, 3.0, 30.0]))
    return kind, order, M, L, ly, d, bw, amp, off


def main():
    n_cases = int(sys.argv[1])
    r = np.random.default_rng(int(sys.argv[2]))
    dev = torch.device("cuda", 0)
    for c in range(n_cases):
        kind, order, M, L, ly, d, bw, amp, off = case(r)
        kw = {"bandwidth": bw} if kind != "linear" else {"scale": 1.0}
        cfg = KernelConfig(static=StaticKernelSpec(kind=kind, **kw), n_levels=M, order=order)
        path = execution_path(L, ly, d, cfg)
        if path == "fp64":
            continue
        n = 3 if max(L, ly) <= 600 else 2
        X = amp * O.gen_brownian(n, L, d, c, ("x",)) + off
        Y = amp * O.gen_brownian(n, ly, d, c, ("y",)) + off
        sp = O.static_params(kind, **kw)
        t0 = time.time()
        R = O.gram_levels(sp, X, Y, M, order)
        SX = O.self_levels(sp, X, M, order)
        SY = O.self_levels(sp, Y, M, order)
        Xt = torch.from_numpy(X).to(dev)
        Yt = torch.from_numpy(Y).to(dev)
        try:
            _, lv = gram_block(Xt, Yt, cfg, want_levels=True)
            lv = lv.cpu().numpy()
            gx = _self_levels_t(Xt, cfg, "fp32").cpu().numpy()
            gy = _self_levels_t(Yt, cfg, "fp32").cpu().numpy()
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"error": str(e), "kind": kind, "order": order, "L": L, "ly": ly,
                              "d": d}), flush=True)
            continue
        cs = np.sqrt(np.clip(SX, 0, None)[:, None, :] * np.clip(SY, 0, None)[None, :, :])
        with np.errstate(divide="ignore", invalid="ignore"):
            a = np.where(cs > 0, np.abs(lv - R) / cs, 0.0).max(axis=(0, 1))
            s = np.concatenate([np.where(SX > 0, np.abs(gx - SX) / SX, 0.0),
                                np.where(SY > 0, np.abs(gy - SY) / SY, 0.0)]).max(axis=0)
        # data radius in scaled units (after midrange centring) and mean step
        pts = np.concatenate([X.reshape(-1, d), Y.reshape(-1, d)])
        c0 = 0.5 * (pts.min(0) + pts.max(0))
        rad2 = float(((pts - c0) ** 2).sum(1).max()) / (bw * bw if kind != "linear" else 1.0)
        step = float(np.sqrt((np.diff(X, axis=1) ** 2).sum(-1)).mean()) / (bw if kind != "linear" else 1.0)
        print(json.dumps({"kind": kind, "order": order, "M": M, "L": L, "ly": ly, "d": d, "bw": bw,
                          "amp": amp, "off": off, "path": path, "rad2": rad2, "step": step,
                          "a": a[1:].tolist(), "s": s[1:].tolist(),
                          "cs": cs.min(axis=(0, 1))[1:].tolist(),
                          "oracle_s": time.time() - t0}), flush=True)


if __name__ == "__main__":
    main()
