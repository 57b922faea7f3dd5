"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference is importable only there):

    cd /tmp && PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python /root/repo/tests/golden/make_golden.py

Writes `tests/golden/*.npz`. The GPU box never reads `/root/reference`; the
tests consume only these committed fixtures.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from sigkern import (KernelConfig, SeedStream, StaticKernelSpec, gen_brownian,  # noqa: E402
                     sig_kernel_gram, sig_levels_dp)
from sigkern.kernels import increment_tensor, sig_levels_bruteforce  # noqa: E402
from sigkern.static.kernels import KERNEL_KINDS  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def _cfg_dict(kind, M, p, difference, norm, **static):
    d = dict(kind=kind, n_levels=M, order=p, difference=difference, normalization=norm)
    d.update(static)
    return d


def _run(X, Y, c):
    st = {k: c[k] for k in ("scale", "degree", "gamma", "bandwidth", "alpha") if k in c}
    cfg = KernelConfig(static=StaticKernelSpec(kind=c["kind"], **st), n_levels=c["n_levels"],
                       order=c["order"], difference=c["difference"],
                       normalization=c["normalization"])
    return sig_kernel_gram(X, Y, cfg=cfg)


def small_cases():
    """Randomised small Gram cases across the KernelConfig surface."""
    rng = np.random.default_rng(2501_07145)
    cases = []
    # every static kind, both normalisations where defined, symmetric and cross
    for n, kind in enumerate(KERNEL_KINDS):
        for norm in ("none", "levelwise", "global"):
            Lx, Ly, d = int(rng.integers(3, 9)), int(rng.integers(3, 9)), int(rng.integers(1, 4))
            X = gen_brownian(3, Lx, d, SeedStream(100 + n, (norm,))).data
            Y = gen_brownian(2, Ly, d, SeedStream(200 + n, (norm,))).data
            M = int(rng.integers(1, 5))
            p = int(rng.integers(1, M + 1))
            extra = {}
            if kind == "polynomial":
                extra = dict(scale=0.7, degree=2, gamma=1.0)
            elif kind == "linear":
                extra = dict(scale=1.3)
            else:
                extra = dict(bandwidth=float(rng.uniform(0.6, 1.8)))
            if kind == "rational_quadratic":
                extra["alpha"] = 1.7
            c = _cfg_dict(kind, M, p, True, norm, **extra)
            cases.append(("k_%s_%s_sym" % (kind, norm), X, None, c))
            cases.append(("k_%s_%s_cross" % (kind, norm), X, Y, c))
    # order / level sweep on rbf and linear
    for M in range(0, 7):
        for p in sorted({1, 2, M if M else 1, None} - {0}, key=lambda v: -1 if v is None else v):
            for kind in ("rbf", "linear"):
                X = gen_brownian(3, 7, 2, SeedStream(300 + M, (kind, str(p)))).data
                Y = gen_brownian(4, 6, 2, SeedStream(400 + M, (kind, str(p)))).data
                c = _cfg_dict(kind, M, p, True, "none")
                cases.append((f"mp_{kind}_M{M}_p{p}", X, Y, c))
    # difference=False
    for kind in ("rbf", "linear"):
        X = gen_brownian(3, 5, 2, SeedStream(500)).data
        Y = gen_brownian(2, 4, 2, SeedStream(501)).data
        for p in (1, 2):
            c = _cfg_dict(kind, 3, p, False, "none")
            cases.append((f"nodiff_{kind}_p{p}", X, Y, c))
    # edge cases: one-point sequences, constant sequences, unequal lengths
    X1 = np.concatenate([np.zeros((1, 5, 2)), gen_brownian(2, 5, 2, SeedStream(600)).data])
    cases.append(("edge_constant_levelwise", X1, None, _cfg_dict("rbf", 3, 1, True, "levelwise")))
    X2 = np.random.default_rng(5).standard_normal((2, 1, 2))  # gen_brownian needs L >= 2
    Y2 = gen_brownian(3, 6, 2, SeedStream(602)).data
    cases.append(("edge_one_point", X2, Y2, _cfg_dict("rbf", 3, 1, True, "none")))
    X3 = gen_brownian(4, 33, 3, SeedStream(603)).data
    Y3 = gen_brownian(5, 70, 3, SeedStream(604)).data
    cases.append(("edge_unequal_len", X3, Y3, _cfg_dict("rbf", 4, 1, True, "levelwise")))
    cases.append(("edge_unequal_len_rev", Y3, X3, _cfg_dict("rbf", 4, 2, True, "none")))
    return cases


BENCH = {
    # name: (k, L, d, M, p, kind, norm, symmetric)
    "c1": (64, 50, 3, 5, 1, "rbf", "levelwise", True),
    "c2": (4, 128, 8, 5, 5, "rbf", "none", False),
    "c2n": (4, 128, 8, 5, 5, "rbf", "levelwise", False),
    "c3": (4, 256, 16, 5, 1, "rbf", "levelwise", False),
    "c3u": (4, 256, 16, 5, 1, "rbf", "none", False),
    "c4": (3, 128, 128, 3, 1, "linear", "none", False),
    "c5": (2, 2048, 4, 8, 1, "rbf", "none", False),
    "c5n": (2, 2048, 4, 8, 1, "rbf", "levelwise", False),
}


def bench_cases():
    out = []
    for name, (k, L, d, M, p, kind, norm, sym) in BENCH.items():
        X = gen_brownian(k, L, d, SeedStream(1)).data
        Y = None if sym else gen_brownian(k, L, d, SeedStream(2)).data
        c = _cfg_dict(kind, M, p, True, norm)
        out.append(("bench_" + name, X, Y, c))
    return out


def main():
    # 1) generator: gen_brownian bits (prefix stability is checked in tests)
    gb = {}
    for (n, L, d, seed) in ((3, 10, 5, 1), (2, 256, 16, 1), (2, 256, 16, 2), (1, 2, 1, 7)):
        gb[f"n{n}_L{L}_d{d}_s{seed}"] = gen_brownian(n, L, d, SeedStream(seed)).data
    gb["child_path"] = gen_brownian(2, 12, 2, SeedStream(31, ("a", "b"))).data
    np.savez(os.path.join(HERE, "brownian.npz"), **gb)

    # 2) Gram cases
    arrays, meta = {}, []
    for name, X, Y, c in small_cases() + bench_cases():
        K = _run(X, Y, c)
        arrays[name + "__X"] = X
        if Y is not None:
            arrays[name + "__Y"] = Y
        arrays[name + "__K"] = K
        meta.append(dict(name=name, cfg=c, symmetric=Y is None))
    arrays["__meta__"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "gram_cases.npz"), **arrays)

    # 3) level recursion on given increment matrices (sig_levels_dp / bruteforce)
    rng = np.random.default_rng(16)
    lv = {}
    for t in range(24):
        T1, T2 = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        M = int(rng.integers(0, 5))
        p = int(rng.integers(1, 4))
        A = rng.standard_normal((T1, T2))
        lv[f"dp{t}__A"] = A
        lv[f"dp{t}__Mp"] = np.array([M, p])
        lv[f"dp{t}__dp"] = sig_levels_dp(A, M, order=p)
        lv[f"dp{t}__bf"] = sig_levels_bruteforce(A, M, order=p)
    mats = [rng.standard_normal((3, 4)) for _ in range(3)]
    lv["perlevel__A"] = np.stack(mats)
    lv["perlevel__dp"] = sig_levels_dp(mats, 3, order=2)
    B = rng.standard_normal((2, 3, 6, 5))
    lv["batched__A"] = B
    lv["batched__dp"] = sig_levels_dp(B, 4, order=2)
    # increment tensors (kernels.py:263-281) for every kind
    for kind in KERNEL_KINDS:
        spec = StaticKernelSpec(kind=kind, bandwidth=1.2)
        x = rng.standard_normal((5, 3))
        y = rng.standard_normal((4, 3))
        lv[f"inc_{kind}__x"] = x
        lv[f"inc_{kind}__y"] = y
        lv[f"inc_{kind}__A"] = increment_tensor(spec, x, y)
        lv[f"inc_{kind}__G"] = increment_tensor(spec, x, y, difference=False)
    np.savez(os.path.join(HERE, "levels.npz"), **lv)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
