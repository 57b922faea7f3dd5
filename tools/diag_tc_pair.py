"""Block-wise error map of the tcgen05 GEMM (development diagnostic)."""
import ctypes
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_07145_b200 import _native

lib = _native.load()
fn = lib.sk_dev_tc_gemm
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
for M, N, K in [(128, 256, 96), (128, 256, 128), (256, 256, 128), (300, 520, 132), (1000, 77, 128)]:
    g = torch.Generator(device="cpu").manual_seed(1)
    A = torch.randn(M, K, generator=g).cuda()
    B = torch.randn(N, K, generator=g).cuda()
    C = torch.full((N, M), float("nan"), device="cuda")
    scratch = torch.empty(2 * (M + N) * K, device="cuda")
    rc = fn(A.data_ptr(), M, B.data_ptr(), N, K, C.data_ptr(), M, scratch.data_ptr(),
            torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = B.double() @ A.double().T
    err = (C.double() - ref).abs() / (B.double().abs() @ A.double().abs().T)
    print(f"M={M} N={N} K={K} rc={rc}")
    for n0 in range(0, N, 128):
        row = []
        for m0 in range(0, M, 128):
            e = err[n0:n0 + 128, m0:m0 + 128]
            row.append("nan" if torch.isnan(e).any() else f"{float(e.max()):.1e}")
        print(f"  n {n0:4d}: " + " ".join(row))
