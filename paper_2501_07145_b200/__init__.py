"""B200-native truncated signature-kernel Gram (drop-in for the reference's dual DP path).

Public surface mirrors the reference's hot-path exports (sigkern/__init__.py:42-51)
plus the KSig-style `SignatureKernel` facade named by the north star.
"""

from .config import KERNEL_KINDS, KernelConfig, LevelValues, StaticKernelSpec
from .errors import ConfigError, NativeError, NumericError, SigkernError
from .facade import (LinearKernel, Matern12Kernel, Matern32Kernel, Matern52Kernel,
                     PolynomialKernel, RationalQuadraticKernel, RBFKernel, SignatureKernel,
                     StaticKernel)
from .features import SigFeatureConfig, fit_sig_features, rfsf_exact_gram
from .kernels import (increment_tensor, self_levels, sig_kernel_dp, sig_kernel_gram,
                      sig_levels_dp, sig_pde_kernel, uses_fast_path)
from .sequences import SeedStream, SequenceBatch, gen_brownian
from .static_kernels import median_heuristic
from .utils import ResourceCounters

__version__ = "0.1.0"

__all__ = [
    "KERNEL_KINDS", "KernelConfig", "LevelValues", "StaticKernelSpec",
    "ConfigError", "NativeError", "NumericError", "SigkernError",
    "StaticKernel", "LinearKernel", "PolynomialKernel", "RBFKernel", "Matern12Kernel",
    "Matern32Kernel", "Matern52Kernel", "RationalQuadraticKernel", "SignatureKernel",
    "increment_tensor", "self_levels", "sig_kernel_dp", "sig_kernel_gram", "sig_levels_dp", "sig_pde_kernel",
    "uses_fast_path", "median_heuristic", "SeedStream", "SequenceBatch", "gen_brownian", "ResourceCounters",
    "SigFeatureConfig", "fit_sig_features", "rfsf_exact_gram", "__version__",
]
