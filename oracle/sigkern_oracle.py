"""CPU oracle for the truncated signature-kernel Gram path — TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference's dual
dynamic-programming path (`/root/reference/pkg/src/sigkern/kernels.py`,
`static/kernels.py`, `sequences.py`, `rng.py`). It exists to CHECK the CUDA
implementation in `paper_2501_07145_b200` and to time the reference algorithm
on host cores (`bench.py`'s `cpu_baseline` leg and `--impl reference`). Only
`tests/`, `__graft_entry__.smoke()` and `bench.py` may import it; the product
package never does, and it is never the thing measured as the product.

Parity pinning: every function below is checked against golden vectors that
were produced by importing the reference itself in the build container
(`tests/golden/make_golden.py` -> `tests/golden/*.npz`; see
`tests/test_oracle_golden.py`). The DP agrees with the reference bitwise on
those vectors (same float64 operation order for the cumulative sums).

Citations are `file:line` into `/root/reference/pkg/src/sigkern/`.
"""

from __future__ import annotations

import hashlib
import math
import os
from concurrent.futures import ThreadPoolExecutor
from itertools import combinations_with_replacement

import numpy as np

KINDS = ("linear", "polynomial", "rbf", "matern12", "matern32", "matern52",
         "rational_quadratic")  # static/kernels.py:25-33


# ---------------------------------------------------------------------------
# inputs: hierarchical Philox streams and Brownian sequences
# ---------------------------------------------------------------------------

def _label_key(label: str) -> tuple[int, int]:
    """64-bit blake2b digest of a label as two uint32 spawn-key words (rng.py:19-23)."""
    v = int.from_bytes(hashlib.blake2b(label.encode("utf-8"), digest_size=8).digest(),
                       "little")
    return v & 0xFFFFFFFF, v >> 32


def philox_generator(seed: int, path: tuple = ()) -> np.random.Generator:
    """Generator of the stream (seed, path) (rng.py:36-57)."""
    key = []
    for label in path:
        key.extend(_label_key(label))
    ss = np.random.SeedSequence(entropy=int(seed), spawn_key=tuple(key))
    return np.random.Generator(np.random.Philox(ss))


def gen_brownian(n: int, length: int, dim: int, seed: int, path: tuple = (),
                 start: int = 0) -> np.ndarray:
    """Random walks from the origin, N(0, 1/(length-1)) steps (sequences.py:110-137).

    Sequence i draws from child stream `seq{i}` of (seed, path), so any
    index window [start, start+n) equals the same rows of a larger batch.
    """
    scale = math.sqrt(1.0 / (length - 1))
    out = np.zeros((n, length, dim))
    for k in range(n):
        g = philox_generator(seed, tuple(path) + (f"seq{start + k}",))
        steps = g.standard_normal((length - 1, dim)) * scale
        np.cumsum(steps, axis=0, out=out[k, 1:, :])
    return out


# ---------------------------------------------------------------------------
# static kernel and increment matrices
# ---------------------------------------------------------------------------

def _static_from_inner(kind, p, inner):
    # static/kernels.py:68-71
    if kind == "linear":
        return p["scale"] * inner
    return (p["scale"] * inner + p["gamma"]) ** p["degree"]


def _static_from_sqdist(kind, p, sq):
    # static/kernels.py:74-89
    bw = p["bandwidth"]
    if kind == "rbf":
        return np.exp(sq / (-2.0 * bw * bw))
    if kind == "rational_quadratic":
        return (1.0 + sq / (2.0 * p["alpha"] * bw * bw)) ** (-p["alpha"])
    r = np.sqrt(sq) / bw
    if kind == "matern12":
        return np.exp(-r)
    if kind == "matern32":
        return (1.0 + math.sqrt(3.0) * r) * np.exp(-math.sqrt(3.0) * r)
    if kind == "matern52":
        return (1.0 + math.sqrt(5.0) * r + (5.0 / 3.0) * r * r) * np.exp(-math.sqrt(5.0) * r)
    raise ValueError(kind)


def static_params(kind="rbf", scale=1.0, degree=3, gamma=1.0, bandwidth=1.0, alpha=1.0):
    """Parameter bundle mirroring StaticKernelSpec (static/kernels.py:39-53)."""
    if kind not in KINDS:
        raise ValueError(kind)
    return dict(kind=kind, scale=float(scale), degree=int(degree), gamma=float(gamma),
                bandwidth=float(bandwidth), alpha=float(alpha))


def point_gram(sp, X, Y):
    """k(x_a, y_b) over the last two axes (kernels.py:252-260)."""
    kind = sp["kind"]
    XY = X @ np.swapaxes(Y, -1, -2)
    if kind in ("linear", "polynomial"):
        return _static_from_inner(kind, sp, XY)
    nx = np.einsum("...ak,...ak->...a", X, X)
    ny = np.einsum("...bk,...bk->...b", Y, Y)
    sq = nx[..., :, None] + ny[..., None, :] - 2.0 * XY
    np.maximum(sq, 0.0, out=sq)
    return _static_from_sqdist(kind, sp, sq)


def pde_kernel(sp, x, y, difference=True):
    """Goursat-PDE value of one pair (kernels.py:334-402), row-streamed restatement:
    K(0,.) = K(.,0) = 1; K(k,l) = both - K(k-1,l-1) + 0.5*C*both, both = K(k,l-1) + K(k-1,l),
    C the double-differenced (or raw, difference=False) point kernel of cell (k-1, l-1)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    C = increments(sp, x, y, difference)
    if difference and (x.shape[0] < 2 or y.shape[0] < 2):
        raise ValueError("pde kernel needs at least one increment per sequence")
    T1, T2 = C.shape
    prev = np.ones(T2 + 1)
    for k in range(1, T1 + 1):
        cur = np.ones(T2 + 1)
        for l in range(1, T2 + 1):
            both = cur[l - 1] + prev[l]
            cur[l] = both - prev[l - 1] + 0.5 * C[k - 1, l - 1] * both
        prev = cur
    return float(prev[T2])


def pde_gram(X, Y=None, sp=None, difference=True, normalization="none"):
    """Gram of pde_kernel values (kernels.py:476-507, 559-571); small inputs only."""
    sp = sp or static_params("rbf")
    Yv = X if Y is None else Y
    K = np.array([[pde_kernel(sp, a, b, difference) for b in Yv] for a in X])
    if normalization == "global":
        sx = np.array([pde_kernel(sp, a, a, difference) for a in X])
        sy = sx if Y is None else np.array([pde_kernel(sp, b, b, difference) for b in Yv])
        K = K / np.sqrt(sx[:, None] * sy[None, :])
    return K


def median_heuristic(X, max_pairs=1_000_000):
    """Median pairwise distance over a deterministic subsample (static/kernels.py:165-187)."""
    X = np.atleast_2d(np.asarray(X, dtype=np.float64))
    n = X.shape[0]
    if n < 2:
        raise ValueError(f"median_heuristic needs at least 2 vectors, got {n}")
    if n * (n - 1) // 2 > max_pairs:
        m = max(2, min(n, int((1.0 + math.sqrt(1.0 + 8.0 * max_pairs)) / 2.0)))
        X = X[np.unique((np.arange(m, dtype=np.int64) * n) // m)]
        n = X.shape[0]
    xx = np.einsum("ij,ij->i", X, X)
    sq = np.maximum(xx[:, None] + xx[None, :] - 2.0 * (X @ X.T), 0.0)  # static/kernels.py:108-114
    med = float(np.median(np.sqrt(sq[np.triu_indices(n, k=1)])))
    return med if med > 0.0 else 1.0


def increments(sp, X, Y, difference=True):
    """Double-differenced point Gram, (..., L1-1, L2-1) (kernels.py:263-281)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    G = point_gram(sp, X, Y)
    if not difference:
        return G
    if X.shape[-2] < 2 or Y.shape[-2] < 2:
        return np.zeros(G.shape[:-2] + (max(X.shape[-2] - 1, 0), max(Y.shape[-2] - 1, 0)))
    return G[..., 1:, 1:] - G[..., :-1, 1:] - G[..., 1:, :-1] + G[..., :-1, :-1]


# ---------------------------------------------------------------------------
# level recursion
# ---------------------------------------------------------------------------

def _excl(a, axis):
    """Exclusive running sum along `axis` (kernels.py:114-126)."""
    c = np.cumsum(a, axis=axis)
    out = np.zeros_like(c)
    n = a.shape[axis]
    dst = [slice(None)] * a.ndim
    src = [slice(None)] * a.ndim
    dst[axis] = slice(1, n)
    src[axis] = slice(0, n - 1)
    out[tuple(dst)] = c[tuple(src)]
    return out


def levels_dp(mats, M: int, p: int = 1) -> np.ndarray:
    """Kiraly-Oberhauser cumulative-sum DP (kernels.py:144-201).

    mats: one (..., T1, T2) increment array or a list of M arrays (level m
    uses mats[m-1], kernels.py:129-141). Returns (..., M+1) with [..., 0] = 1.
    State R[q, r] holds weighted products of index pairs ending at (i, j)
    whose trailing multiplicities are (q+1, r+1).
    """
    M = int(M)
    if isinstance(mats, (list, tuple)):
        if M >= 1 and len(mats) != M:
            raise ValueError(
                f"per-level increment list must have n_levels={M} entries, got {len(mats)}")
        per = [np.asarray(a, dtype=np.float64) for a in mats]
        if M >= 1 and len({a.shape for a in per}) > 1:
            raise ValueError("per-level increment matrices disagree on shape")
        first = per[0] if per else np.zeros((0, 0))
        pick = lambda m: per[m - 1]
    else:
        first = np.asarray(mats, dtype=np.float64)
        pick = lambda m: first
    if first.ndim < 2:
        first = first.reshape((0, 0))
    lead = first.shape[:-2]
    out = np.zeros(lead + (M + 1,))
    out[..., 0] = 1.0
    if M == 0 or first.shape[-1] == 0 or first.shape[-2] == 0:
        return out
    p = max(1, min(int(p), M))
    R = np.zeros((p, p) + first.shape)
    R[0, 0] = pick(1)
    out[..., 1] = R[0, 0].sum(axis=(-1, -2))
    for m in range(2, M + 1):
        A = pick(m)
        nxt = np.zeros_like(R)
        tot = R.sum(axis=(0, 1))
        nxt[0, 0] = A * _excl(_excl(tot, -1), -2)
        if p > 1:
            rows = R.sum(axis=1)   # SX[q] = sum_r R[q, r]
            cols = R.sum(axis=0)   # SY[r] = sum_q R[q, r]
            for q in range(1, p):
                nxt[q, 0] = (A / (q + 1)) * _excl(rows[q - 1], -1)
                nxt[0, q] = (A / (q + 1)) * _excl(cols[q - 1], -2)
            for q in range(1, p):
                for r in range(1, p):
                    nxt[q, r] = (A / ((q + 1) * (r + 1))) * R[q - 1, r - 1]
        R = nxt
        out[..., m] = R.sum(axis=(0, 1, -1, -2))
    return out


def _multi_index_weight(idx, p):
    # 1/prod(n_b!) over runs, 0 if a run exceeds p (kernels.py:204-215)
    w, run = 1.0, 1
    for a in range(1, len(idx)):
        if idx[a] == idx[a - 1]:
            run += 1
            if run > p:
                return 0.0
            w /= run
        else:
            run = 1
    return w


def levels_bruteforce(mats, M: int, p: int = 1) -> np.ndarray:
    """Enumerate nondecreasing multi-index pairs (kernels.py:218-249). Tiny inputs only."""
    M = int(M)
    out = np.zeros(M + 1)
    out[0] = 1.0
    if M == 0:
        return out
    per = ([np.asarray(a, dtype=np.float64) for a in mats]
           if isinstance(mats, (list, tuple)) else [np.asarray(mats, dtype=np.float64)] * M)
    T1, T2 = per[0].shape[-2:]
    if T1 == 0 or T2 == 0:
        return out
    p = max(1, min(int(p), M))
    for m in range(1, M + 1):
        acc = 0.0
        for ii in combinations_with_replacement(range(T1), m):
            wi = _multi_index_weight(ii, p)
            if wi == 0.0:
                continue
            for jj in combinations_with_replacement(range(T2), m):
                wj = _multi_index_weight(jj, p)
                if wj == 0.0:
                    continue
                prod = wi * wj
                for a in range(m):
                    prod *= per[a][ii[a], jj[a]]
                acc += prod
        out[m] = acc
    return out


# ---------------------------------------------------------------------------
# Gram driver and normalisation
# ---------------------------------------------------------------------------

_STATE_ARRAYS = 6  # kernels.py:56


def _tile_side(Lx, Ly, p, difference, tile_memory):
    # kernels.py:439-445
    T1 = Lx - 1 if difference else Lx
    T2 = Ly - 1 if difference else Ly
    per_pair = 8 * (Lx * Ly + (2 * p * p + _STATE_ARRAYS) * max(T1 * T2, 1))
    return max(1, int(math.isqrt(max(1, int(tile_memory) // per_pair))))


def gram_levels(sp, X, Y, M, p, difference=True, symmetric=False, n_threads=1,
                tile_memory=256 * 2 ** 20):
    """(Nx, Ny, M+1) level values over fixed pair tiles (kernels.py:437-473)."""
    p = max(1, min(int(p), M)) if M >= 1 else 1
    Nx, Ny = X.shape[0], Y.shape[0]
    b = _tile_side(X.shape[1], Y.shape[1], p, difference, tile_memory)
    out = np.empty((Nx, Ny, M + 1))
    jobs = [(i0, min(i0 + b, Nx), j0, min(j0 + b, Ny))
            for bi, i0 in enumerate(range(0, Nx, b))
            for bj, j0 in enumerate(range(0, Ny, b))
            if not (symmetric and bj < bi)]

    def run(job):
        i0, i1, j0, j1 = job
        A = increments(sp, X[i0:i1, None], Y[None, j0:j1], difference)
        t = levels_dp(A, M, p)
        if symmetric and i0 == j0:  # bitwise mirror (kernels.py:429-434)
            for m in range(t.shape[-1]):
                u = np.triu(t[..., m])
                t[..., m] = u + np.triu(t[..., m], 1).T
        out[i0:i1, j0:j1] = t
        if symmetric and j0 > i0:
            out[j0:j1, i0:i1] = t.transpose(1, 0, 2)

    if n_threads <= 1 or len(jobs) <= 1:
        for job in jobs:
            run(job)
    else:
        with ThreadPoolExecutor(max_workers=n_threads) as pool:
            list(pool.map(run, jobs))
    return out


def self_levels(sp, X, M, p, difference=True):
    """Per-sequence self level values via the paired increments (kernels.py:589-595)."""
    A = increments(sp, X, X, difference)
    return levels_dp(A, M, max(1, min(int(p), M)) if M >= 1 else 1)


def normalize_levelwise(levels, dx, dy):
    # kernels.py:510-516
    M = levels.shape[-1] - 1
    den = np.sqrt(np.clip(dx, 0.0, None)[:, None, :] * np.clip(dy, 0.0, None)[None, :, :])
    terms = np.divide(levels, den, out=np.zeros_like(levels), where=den > 0)
    return terms.sum(axis=-1) / (M + 1)


def normalize_global(K, sx, sy):
    # kernels.py:519-527
    bad_x = np.flatnonzero(sx <= 0)
    bad_y = np.flatnonzero(sy <= 0)
    if bad_x.size or bad_y.size:
        which = bad_x if bad_x.size else bad_y
        raise ArithmeticError(
            f"global normalization undefined: non-positive self-kernel for "
            f"input sequence index {int(which[0])}")
    return K / np.sqrt(sx[:, None] * sy[None, :])


def gram(X, Y=None, *, sp=None, M=5, p=1, difference=True, normalization="none",
         n_threads=1, tile_memory=256 * 2 ** 20):
    """Signature-kernel Gram matrix, algorithm="dp" (kernels.py:530-600)."""
    sp = sp or static_params()
    X = np.asarray(X, dtype=np.float64)
    symmetric = Y is None
    Y = X if symmetric else np.asarray(Y, dtype=np.float64)
    p_eff = 1 if M == 0 else max(1, min(int(p if p is not None else M), M))
    lv = gram_levels(sp, X, Y, M, p_eff, difference, symmetric, n_threads, tile_memory)
    if normalization == "none":
        return lv.sum(axis=-1)
    dx = self_levels(sp, X, M, p_eff, difference)
    dy = dx if symmetric else self_levels(sp, Y, M, p_eff, difference)
    if normalization == "levelwise":
        return normalize_levelwise(lv, dx, dy)
    return normalize_global(lv.sum(axis=-1), dx.sum(axis=-1), dy.sum(axis=-1))


# --- rfsf_exact_gram (features.py:397-475) -----------------------------------

def static_features(slot, X):
    """transform_static_features (static/features.py:102-124) of a fitted slot,
    given as a dict: kind ("rff"/"rff1d"/"nystroem"), n_components, weights,
    phases, landmarks, whiten, base (static_params of the nystroem base kernel)."""
    X = np.asarray(X, dtype=np.float64)
    D = int(slot["n_components"])
    if slot["kind"] == "rff":
        P = X @ slot["weights"]
        s = 1.0 / math.sqrt(D)
        return np.concatenate([s * np.cos(P), s * np.sin(P)], axis=-1)
    if slot["kind"] == "rff1d":
        return math.sqrt(2.0 / D) * np.cos(X @ slot["weights"] + slot["phases"])
    lead = X.shape[:-1]
    K = point_gram(slot["base"], X.reshape(-1, X.shape[-1]), slot["landmarks"])
    return (K @ slot["whiten"]).reshape(*lead, slot["whiten"].shape[1])


def lifted_levels(slots, Xa, Xb, M, p, difference=True):
    """_lifted_level_grams (features.py:397-424): level m's increments come from
    slot m's feature inner products. -> (Na, Nb, M+1)."""
    Na, La = Xa.shape[:2]
    Nb, Lb = Xb.shape[:2]
    if M == 0:
        return np.ones((Na, Nb, 1))
    mats = []
    for slot in slots:
        Ux = static_features(slot, Xa)
        Uy = static_features(slot, Xb)
        G = (Ux.reshape(Na * La, -1) @ Uy.reshape(Nb * Lb, -1).T).reshape(
            Na, La, Nb, Lb).transpose(0, 2, 1, 3)
        mats.append(G[..., 1:, 1:] - G[..., :-1, 1:] - G[..., 1:, :-1] + G[..., :-1, :-1]
                    if difference else G)
    return levels_dp(mats, M, p)


def lifted_self_levels(slots, Xa, M, p, difference=True):
    """_lifted_self_levels (features.py:427-443). -> (N, M+1)."""
    if M == 0:
        return np.ones((Xa.shape[0], 1))
    mats = []
    for slot in slots:
        U = static_features(slot, Xa)
        G = U @ U.transpose(0, 2, 1)
        mats.append(G[..., 1:, 1:] - G[..., :-1, 1:] - G[..., 1:, :-1] + G[..., :-1, :-1]
                    if difference else G)
    return levels_dp(mats, M, p)


def rfsf_exact_gram(slots, X, Y=None, M=None, p=1, difference=True, normalize=False):
    """rfsf_exact_gram (features.py:446-475) from fitted slot dicts."""
    M = len(slots) if M is None else M
    Xa = np.asarray(X, dtype=np.float64)
    sym = Y is None
    Xb = Xa if sym else np.asarray(Y, dtype=np.float64)
    levels = lifted_levels(slots, Xa, Xb, M, p, difference)
    if not normalize:
        K = levels.sum(axis=-1)
    else:
        if sym:
            dx = dy = np.einsum("iim->im", levels).copy()
        else:
            dx = lifted_self_levels(slots, Xa, M, p, difference)
            dy = lifted_self_levels(slots, Xb, M, p, difference)
        K = normalize_levelwise(levels, dx, dy)
    if sym:
        K = np.triu(K) + np.triu(K, 1).T
    return K


def host_threads() -> int:
    return len(os.sched_getaffinity(0))
