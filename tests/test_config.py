"""Host-side boundary logic (no device needed): configuration validation and
messages mirror the reference (kernels.py:59-91, static/kernels.py:39-65),
the KSig facade maps onto KernelConfig, and compute entry points refuse to run
without CUDA instead of falling back to the CPU."""

import numpy as np
import pytest
import torch

from paper_2501_07145_b200 import (ConfigError, KernelConfig, LevelValues, LinearKernel,
                                   RBFKernel, ResourceCounters, SignatureKernel,
                                   StaticKernelSpec, sig_kernel_gram)
from paper_2501_07145_b200.utils import dp_flops


class TestKernelConfig:  # test_kernels.py:40-64
    def test_defaults(self):
        cfg = KernelConfig()
        assert (cfg.n_levels, cfg.order, cfg.difference) == (5, 1, True)
        assert cfg.normalization == "none"

    def test_effective_order(self):
        assert KernelConfig(n_levels=4, order=None).effective_order == 4
        assert KernelConfig(n_levels=3, order=7).effective_order == 3
        assert KernelConfig(n_levels=3, order=2).effective_order == 2
        assert KernelConfig(n_levels=0, order=None).effective_order == 1

    def test_validation(self):
        with pytest.raises(ValueError, match="n_levels"):
            KernelConfig(n_levels=-1)
        with pytest.raises(ValueError, match="order"):
            KernelConfig(order=0)
        with pytest.raises(ValueError, match="normalization"):
            KernelConfig(normalization="unit")

    def test_level_values_api(self):
        lv = LevelValues([1.0, 2.0, 3.0])
        assert lv.n_levels == 2 and lv.total() == 6.0 and lv[1] == 2.0


class TestStaticSpec:  # static/kernels.py:55-65
    def test_validation(self):
        with pytest.raises(ValueError, match="unknown kernel kind"):
            StaticKernelSpec(kind="cosine")
        for kw, word in ((dict(scale=0), "scale"), (dict(degree=0), "degree"),
                         (dict(bandwidth=-1), "bandwidth"), (dict(alpha=0), "alpha")):
            with pytest.raises(ValueError, match=word):
                StaticKernelSpec(**kw)


class TestFacade:
    def test_mapping(self):
        k = SignatureKernel(n_levels=4, order=7, normalize=True, static_kernel=RBFKernel(2.0))
        assert k.config.normalization == "levelwise"
        assert k.order == 4 and k.n_levels == 4
        assert k.config.static == StaticKernelSpec(kind="rbf", bandwidth=2.0)
        k2 = SignatureKernel(normalize=False, static_kernel=LinearKernel(0.5))
        assert k2.config.normalization == "none" and k2.config.static.scale == 0.5
        assert SignatureKernel(normalization="global").config.normalization == "global"


class TestBoundaryErrors:  # test_kernels.py:367-373, 435-438
    def test_unknown_algorithm(self):
        with pytest.raises(ValueError, match="algorithm"):
            sig_kernel_gram(np.zeros((2, 3, 2)), algorithm="magic")

    def test_pde_rejects_levelwise(self):
        with pytest.raises(ConfigError, match="levelwise"):
            sig_kernel_gram(np.zeros((2, 3, 2)), cfg=KernelConfig(normalization="levelwise"),
                            algorithm="pde")

    @pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
    def test_no_cpu_fallback(self):
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            sig_kernel_gram(np.zeros((2, 3, 2)))


def test_flop_counter_matches_reference_formula():
    # one pair, T1 = T2 = 2, M = 2, p = 1: increment_tensor 3*3*d + 3*2*2 (kernels.py:273-280)
    # plus sig_levels_dp cell + (1+3)*cell + 1*cell (kernels.py:178-199)
    assert dp_flops(1, 2, 2, 1, 2, 1, True) == 9 + 12 + 4 + 16 + 4
    c = ResourceCounters()
    c.add_flops(5)
    c.observe_bytes(7)
    c2 = ResourceCounters()
    c2.observe_bytes(9)
    c.merge(c2)
    assert (c.flops, c.peak_bytes) == (5, 9)
