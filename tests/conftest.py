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
