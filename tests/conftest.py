import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class GramCases:
    """Golden Gram cases produced by the reference (tests/golden/make_golden.py)."""

    def __init__(self):
        self.z = np.load(os.path.join(GOLDEN, "gram_cases.npz"))
        self.meta = json.loads(bytes(self.z["__meta__"]).decode())

    def __iter__(self):
        for m in self.meta:
            name = m["name"]
            X = self.z[name + "__X"]
            Y = None if m["symmetric"] else self.z[name + "__Y"]
            yield name, X, Y, m["cfg"], self.z[name + "__K"]

    def get(self, name):
        for case in self:
            if case[0] == name:
                return case
        raise KeyError(name)


@pytest.fixture(scope="session")
def gram_cases():
    return GramCases()


@pytest.fixture(scope="session")
def levels_golden():
    return np.load(os.path.join(GOLDEN, "levels.npz"))


@pytest.fixture(scope="session")
def brownian_golden():
    return np.load(os.path.join(GOLDEN, "brownian.npz"))


def oracle_static(c):
    from oracle import sigkern_oracle as O
    keys = ("scale", "degree", "gamma", "bandwidth", "alpha")
    return O.static_params(c["kind"], **{k: c[k] for k in keys if k in c})


def pkg_config(c):
    from paper_2501_07145_b200 import KernelConfig, StaticKernelSpec
    keys = ("scale", "degree", "gamma", "bandwidth", "alpha")
    spec = StaticKernelSpec(kind=c["kind"], **{k: c[k] for k in keys if k in c})
    return KernelConfig(static=spec, n_levels=c["n_levels"], order=c["order"],
                        difference=c["difference"], normalization=c["normalization"])


class RfsfCase:
    """One rfsf_exact_gram golden case (tests/golden/make_rfsf_golden.py)."""

    def __init__(self, z, name):
        import ast
        g = lambda k: z[f"{name}__{k}"]  # noqa: E731
        self.name = name
        self.X = g("X")
        self.Y = z[f"{name}__Y"] if f"{name}__Y" in z.files else None
        self.K = g("K")
        self.direct = z[f"{name}__direct"] if f"{name}__direct" in z.files else None
        D, M, order, diff, norm, sym = [int(v) for v in g("meta")]
        self.D, self.M, self.order = D, M, (None if order < 0 else order)
        self.difference, self.normalize, self.sym = bool(diff), bool(norm), bool(sym)
        self.kind = str(g("kind"))
        self.base = ast.literal_eval(str(g("base")))
        self.slots = []
        for a in range(M):
            s = {"kind": self.kind, "n_components": D}
            for f in ("weights", "phases", "landmarks", "whiten"):
                key = f"{name}__slot{a}__{f}"
                s[f] = z[key] if key in z.files else None
            self.slots.append(s)

    @property
    def p(self):
        if self.M == 0:
            return 1
        return self.M if self.order is None else min(self.order, self.M)

    def oracle_slots(self):
        from oracle import sigkern_oracle as O
        base = O.static_params(**self.base) if self.kind == "nystroem" else None
        return [dict(s, base=base) for s in self.slots]

    def state(self):
        """The case's fitted map as the package's mirror types."""
        from paper_2501_07145_b200.config import StaticKernelSpec
        from paper_2501_07145_b200.features import (SigFeatureConfig, SigFeatureState,
                                                    StaticFeatureSpec, StaticFeatureState)
        spec = StaticFeatureSpec(kind=self.kind, n_components=self.D,
                                 base_kernel=StaticKernelSpec(**self.base))
        cfg = SigFeatureConfig(variant="rfsf_full", static=spec, n_components=self.D,
                               projection=self.D, n_levels=self.M, order=self.order,
                               difference=self.difference)
        d = self.X.shape[-1]
        slots = []
        for s in self.slots:
            out = {"rff": 2 * self.D, "rff1d": self.D}.get(self.kind)
            if out is None:
                out = s["whiten"].shape[1]
            slots.append(StaticFeatureState(spec, d, out, s["weights"], s["phases"],
                                            s["landmarks"], s["whiten"]))
        return SigFeatureState(cfg, d, slots, None, [])


@pytest.fixture(scope="session")
def rfsf_cases():
    z = np.load(os.path.join(GOLDEN, "rfsf.npz"))
    names = sorted({k.split("__")[0] for k in z.files})
    return [RfsfCase(z, n) for n in names]
