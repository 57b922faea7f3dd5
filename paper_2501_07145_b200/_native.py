"""ctypes binding of the C ABI in include/sigkern_b200.h (libsigkern_b200.so).

The library is built in-tree (`make`, or `__graft_entry__.build()`); there is
no CPU fallback — if the library or a CUDA device is missing, every compute
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SK_LIB_OVERRIDE: development A/B timing of alternative builds of the same library
LIB_PATH = os.environ.get("SK_LIB_OVERRIDE") or os.path.join(_HERE, "_lib", "libsigkern_b200.so")

SK_OK, SK_ERR_INVALID, SK_ERR_CUDA, SK_ERR_WORKSPACE, SK_ERR_UNSUPPORTED = range(5)
KIND_CODES = {"linear": 0, "polynomial": 1, "rbf": 2, "matern12": 3, "matern32": 4,
              "matern52": 5, "rational_quadratic": 6}
NORM_CODES = {"none": 0, "levelwise": 1, "global": 2}
PREC_CODES = {"fp32": 0, "fp64": 1}

# every symbol include/sigkern_b200.h declares
EXPORTS = ("sk_abi_version", "sk_last_error", "sk_workspace_bytes", "sk_fast_path",
           "sk_self_levels", "sk_gram", "sk_levels_dp_workspace_bytes", "sk_levels_dp",
           "sk_increment_tensor", "sk_pairwise_dist", "sk_pde_workspace_bytes", "sk_pde_gram",
           "sk_pde_self", "sk_static_features_workspace_bytes", "sk_static_features",
           "sk_lifted_workspace_bytes", "sk_lifted_gram_workspace_bytes", "sk_lifted_gram",
           "sk_lifted_self_levels")


class SkStaticSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("degree", ctypes.c_int32),
                ("scale", ctypes.c_double), ("gamma", ctypes.c_double),
                ("bandwidth", ctypes.c_double), ("alpha", ctypes.c_double)]


class SkKernelConfig(ctypes.Structure):
    _fields_ = [("static_spec", SkStaticSpec), ("n_levels", ctypes.c_int32),
                ("order", ctypes.c_int32), ("difference", ctypes.c_int32),
                ("normalization", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("flags", ctypes.c_int32)]


class SkFeatureMap(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("n_components", ctypes.c_int64), ("out_dim", ctypes.c_int64),
                ("weights", ctypes.c_void_p), ("phases", ctypes.c_void_p),
                ("landmarks", ctypes.c_void_p), ("whiten", ctypes.c_void_p),
                ("base", SkStaticSpec)]


_lock = threading.Lock()
_lib = None


def _declare(lib):
    P, I64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
    CFG = ctypes.POINTER(SkKernelConfig)
    lib.sk_abi_version.restype = ctypes.c_int
    lib.sk_abi_version.argtypes = []
    lib.sk_last_error.restype = ctypes.c_char_p
    lib.sk_last_error.argtypes = []
    lib.sk_workspace_bytes.restype = SZ
    lib.sk_workspace_bytes.argtypes = [I64, I64, I64, I64, I64, CFG]
    lib.sk_fast_path.restype = ctypes.c_int
    lib.sk_fast_path.argtypes = [I64, I64, I64, CFG]
    lib.sk_self_levels.restype = ctypes.c_int
    lib.sk_self_levels.argtypes = [P, I64, I64, I64, CFG, P, P, SZ, P]
    lib.sk_gram.restype = ctypes.c_int
    lib.sk_gram.argtypes = [P, I64, I64, P, I64, I64, I64, I32, CFG, I64, I64, P, P, P, I64,
                            P, P, SZ, P]
    lib.sk_levels_dp_workspace_bytes.restype = SZ
    lib.sk_levels_dp_workspace_bytes.argtypes = [I64, I64, I64, I32, I32]
    lib.sk_levels_dp.restype = ctypes.c_int
    lib.sk_levels_dp.argtypes = [P, I64, I64, I64, I32, I32, I32, P, P, SZ, P]
    SPEC = ctypes.POINTER(SkStaticSpec)
    lib.sk_pde_workspace_bytes.restype = SZ
    lib.sk_pde_workspace_bytes.argtypes = [I64, I64, I32]
    lib.sk_pde_gram.restype = ctypes.c_int
    lib.sk_pde_gram.argtypes = [P, I64, I64, P, I64, I64, I64, I32, SPEC, I32, I64, I64, P, I64,
                                P, SZ, P]
    lib.sk_pde_self.restype = ctypes.c_int
    lib.sk_pde_self.argtypes = [P, I64, I64, I64, SPEC, I32, P, P, SZ, P]
    lib.sk_pairwise_dist.restype = ctypes.c_int
    lib.sk_pairwise_dist.argtypes = [P, I64, I64, P, P]
    FMAP = ctypes.POINTER(SkFeatureMap)
    OFFS = ctypes.POINTER(ctypes.c_int64)
    lib.sk_static_features_workspace_bytes.restype = SZ
    lib.sk_static_features_workspace_bytes.argtypes = [FMAP, I64]
    lib.sk_static_features.restype = ctypes.c_int
    lib.sk_static_features.argtypes = [FMAP, P, I64, I64, P, I64, P, SZ, P]
    lib.sk_lifted_workspace_bytes.restype = SZ
    lib.sk_lifted_workspace_bytes.argtypes = [I64, I64, I32, I32, I32]
    lib.sk_lifted_gram_workspace_bytes.restype = SZ
    lib.sk_lifted_gram_workspace_bytes.argtypes = [I64, I64, I64, I64, I32, I32, I32]
    lib.sk_lifted_gram.restype = ctypes.c_int
    lib.sk_lifted_gram.argtypes = [P, I64, I64, P, I64, I64, I64, OFFS, I32, I32, I32, I32, I32,
                                   I64, I64, P, P, P, I64, P, P, SZ, P]
    lib.sk_lifted_self_levels.restype = ctypes.c_int
    lib.sk_lifted_self_levels.argtypes = [P, I64, I64, I64, OFFS, I32, I32, I32, P, P, SZ, P]
    lib.sk_increment_tensor.restype = ctypes.c_int
    lib.sk_increment_tensor.argtypes = [P, I64, I64, P, I64, I64, I64, I32,
                                        ctypes.POINTER(SkStaticSpec), I32, P, P]


def load():
    """Load (once) and return the CDLL; raises if the library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                    "there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            _declare(lib)
            if lib.sk_abi_version() != 2:  # include/sigkern_b200.h SK_ABI_VERSION
                raise RuntimeError("libsigkern_b200 ABI version mismatch")
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc == SK_OK:
        return
    from .errors import NativeError
    msg = load().sk_last_error().decode(errors="replace")
    if rc == SK_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    raise NativeError(f"{what} failed (code {rc}): {msg}")


def static_struct(spec) -> SkStaticSpec:
    return SkStaticSpec(KIND_CODES[spec.kind], int(spec.degree), float(spec.scale),
                        float(spec.gamma), float(spec.bandwidth), float(spec.alpha))


SK_FLAG_NO_FIXUP = 1  # include/sigkern_b200.h sk_config_flags


def config_struct(cfg, precision: str = "fp32", flags: int = 0) -> SkKernelConfig:
    if precision not in PREC_CODES:
        raise ValueError(f"precision must be one of {tuple(PREC_CODES)}, got {precision!r}")
    return SkKernelConfig(static_struct(cfg.static), int(cfg.n_levels), int(cfg.effective_order),
                          1 if cfg.difference else 0, NORM_CODES[cfg.normalization],
                          PREC_CODES[precision], int(flags))
