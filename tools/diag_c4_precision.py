"""Diagnostics: error sources of the GEMM-fed linear path at c4 shapes (development helper)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sigkern_oracle as O  # noqa: E402
from paper_2501_07145_b200 import KernelConfig, SeedStream, StaticKernelSpec, gen_brownian, sig_kernel_gram  # noqa: E402
from paper_2501_07145_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
X = gen_brownian(n, 128, 128, SeedStream(1)).data
Y = gen_brownian(n, 128, 128, SeedStream(2)).data
cfg = KernelConfig(static=StaticKernelSpec(kind="linear"), n_levels=3)
K = sig_kernel_gram(X, Y, cfg=cfg)
R = O.gram(X, Y, sp=O.static_params("linear"), M=3, p=1)
rel = np.abs(K - R) / np.abs(R)
print("K rel err: max %.3e median %.3e  |R| min %.3g max %.3g" % (rel.max(), np.median(rel), np.abs(R).min(), np.abs(R).max()))
# increment GEMM error (tcgen05 3xTF32 vs exact products of the fp32-rounded increments)
lib = _native.load()
dX = np.diff(X, axis=1).reshape(-1, 128).astype(np.float32)
dY = np.diff(Y, axis=1).reshape(-1, 128).astype(np.float32)
A = torch.from_numpy(dY).cuda(); B = torch.from_numpy(dX).cuda()
M_, N_ = A.shape[0], B.shape[0]
C = torch.empty((N_, M_), dtype=torch.float32, device="cuda")
scratch = torch.empty(2 * (M_ + N_) * 128, dtype=torch.float32, device="cuda")
fn = lib.sk_dev_tc_gemm
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
assert fn(A.data_ptr(), M_, B.data_ptr(), N_, 128, C.data_ptr(), M_, scratch.data_ptr(), None) == 0
torch.cuda.synchronize()
ex = dX.astype(np.float64) @ dY.astype(np.float64).T
sg = (torch.from_numpy(dX).cuda() @ torch.from_numpy(dY).cuda().T).cpu().numpy().astype(np.float64)
tcv = C.cpu().numpy().astype(np.float64)
scale = np.abs(dX.astype(np.float64)) @ np.abs(dY.astype(np.float64)).T
print("A err / sum|ab|: tc max %.3e rms %.3e | torch sgemm max %.3e rms %.3e" % (
    (np.abs(tcv - ex) / scale).max(), np.sqrt(((tcv - ex) / scale) ** 2).mean() ** 0.5 if False else np.sqrt((((tcv - ex) / scale) ** 2).mean()),
    (np.abs(sg - ex) / scale).max(), np.sqrt((((sg - ex) / scale) ** 2).mean())))
# K from exact-f32-input A with a float64 DP (error floor of the inputs)
def levels_from(Afull):
    out = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            a = Afull[i * 127:(i + 1) * 127, j * 127:(j + 1) * 127]
            out[i, j] = O.levels_dp(a, 3, 1).sum()
    return out
for name, Am in (("exact-f32in", ex), ("tc", tcv), ("sgemm", sg)):
    Kx = levels_from(Am)
    print("f64 DP on %-12s A: K max rel %.3e" % (name, (np.abs(Kx - R) / np.abs(R)).max()))
# accumulation-chain test: the same GEMM as 4 (and 16) separate K slices summed in float64
for parts in (4, 16):
    acc = np.zeros_like(ex)
    w = 128 // parts
    for c in range(parts):
        As = A[:, c * w:(c + 1) * w].contiguous(); Bs = B[:, c * w:(c + 1) * w].contiguous()
        Cs = torch.empty((N_, M_), dtype=torch.float32, device="cuda")
        assert fn(As.data_ptr(), M_, Bs.data_ptr(), N_, w, Cs.data_ptr(), M_, scratch.data_ptr(), None) == 0
        torch.cuda.synchronize()
        acc += Cs.cpu().numpy().astype(np.float64)
    print("tc in %2d K-slices summed in f64: err/sum|ab| max %.3e rms %.3e" % (
        parts, (np.abs(acc - ex) / scale).max(), np.sqrt((((acc - ex) / scale) ** 2).mean())))
