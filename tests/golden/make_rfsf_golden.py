"""Golden vectors for rfsf_exact_gram (features.py:446-475), produced by the
REFERENCE itself. Run in the build container:

    cd /tmp && PYTHONPATH=/root/reference/pkg/src python /root/repo/tests/golden/make_rfsf_golden.py

Each case stores the fitted slot parameters (so the device path and the oracle
evaluate the same map), the inputs, the reference's rfsf_exact_gram output
and, for rfsf_full with small widths, the reference's primal
sig_feature_gram (criterion 06: the lifted Gram equals the materialised
feature inner products).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sigkern import SeedStream, StaticKernelSpec, gen_brownian  # noqa: E402
from sigkern.features import (SigFeatureConfig, fit_sig_features, rfsf_exact_gram,  # noqa: E402
                              sig_feature_gram)
from sigkern.static.features import StaticFeatureSpec  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name, static kind, base kernel, D, M, order, difference, normalize, sym, X shape, Y shape
CASES = [
    ("rff_cross", "rff", None, 3, 3, 1, True, False, False, (4, 6, 2), (3, 5, 2)),
    ("rff_sym_norm", "rff", None, 4, 3, 2, True, True, True, (5, 7, 3), None),
    ("rff_geo", "rff", None, 2, 4, None, True, False, False, (3, 5, 2), (4, 6, 2)),
    ("rff_nodiff", "rff", None, 3, 2, 1, False, False, False, (3, 4, 2), (2, 5, 2)),
    ("rff_cross_norm", "rff", None, 3, 3, 3, True, True, False, (3, 6, 2), (4, 5, 2)),
    ("nys_rbf", "nystroem", dict(kind="rbf", bandwidth=1.2), 4, 3, 1, True, False, False,
     (4, 6, 2), (3, 7, 2)),
    ("nys_matern", "nystroem", dict(kind="matern32", bandwidth=0.9), 5, 2, 2, True, True, True,
     (5, 6, 3), None),
    ("nys_linear", "nystroem", dict(kind="linear", scale=0.8), 3, 3, 1, True, False, False,
     (3, 5, 3), (3, 4, 3)),
    ("rff_M1", "rff", None, 3, 1, 1, True, False, False, (3, 5, 2), (2, 4, 2)),
    ("rff_M0", "rff", None, 3, 0, 1, True, False, False, (2, 4, 2), (3, 4, 2)),
    ("rff_long", "rff", None, 6, 5, 1, True, True, False, (3, 40, 3), (2, 33, 3)),
]


def main():
    out = {}
    for (name, kind, base, D, M, order, diff, norm, sym, xs, ys) in CASES:
        X = gen_brownian(*xs, SeedStream(21, (name,))).data
        Y = None if sym else gen_brownian(*ys, SeedStream(22, (name,))).data
        static = StaticFeatureSpec(kind=kind, n_components=D,
                                   base_kernel=StaticKernelSpec(**(base or {})))
        cfg = SigFeatureConfig(variant="rfsf_full", static=static, n_components=D,
                               projection=D, n_levels=M, order=order, difference=diff)
        state = fit_sig_features(cfg, X, SeedStream(23, (name,)))  # fitted on X's points
        K = rfsf_exact_gram(state, X, Y, normalize=norm)
        p = f"{name}__"
        out[p + "X"] = X
        if Y is not None:
            out[p + "Y"] = Y
        out[p + "K"] = K
        out[p + "meta"] = np.array([D, M, -1 if order is None else order, int(diff), int(norm),
                                    int(sym)])
        out[p + "kind"] = np.array(kind)
        out[p + "base"] = np.array(repr(base or {}))
        for a, st in enumerate(state.slot_states):
            q = f"{p}slot{a}__"
            for f in ("weights", "phases", "landmarks", "whiten"):
                v = getattr(st, f)
                if v is not None:
                    out[q + f] = v
        width = int(np.prod([s.out_dim for s in state.slot_states] or [1]))
        if width <= 4096 and M >= 1:
            out[p + "direct"] = sig_feature_gram(state, X, Y, normalize=norm)
    np.savez_compressed(os.path.join(HERE, "rfsf.npz"), **out)
    print(len(out), "arrays")


if __name__ == "__main__":
    main()
