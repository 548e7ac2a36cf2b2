"""Correctness + timing of the warm-path DMMA GEMM (dgemm.cuh) at the large-block sizes, beside
torch's cuBLAS FP64 GEMM on the same device (context).  Usage: python tools/dgemm_probe.py"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_04174_b200 import load_library  # noqa: E402

P = ctypes.POINTER(ctypes.c_double)
L = load_library()
L.sosadmm_debug_dgemm.argtypes = [ctypes.c_int] * 3 + [P, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_int,
                                                       ctypes.POINTER(ctypes.c_float)]


def dp(a):
    return a.ctypes.data_as(P)


def run(M, N, K, tA, up, var=-1, reps=50):
    rng = np.random.default_rng(1)
    A = np.asfortranarray(rng.standard_normal((K, M) if tA else (M, K)))
    B = np.asfortranarray(rng.standard_normal((K, N)))
    C = np.zeros((M, N), order="F")
    ms = ctypes.c_float(0)
    assert L.sosadmm_debug_dgemm(M, N, K, dp(A), tA, up, dp(B), dp(C), var, reps, ctypes.byref(ms)) == 0
    ref = (A.T if tA else A) @ B
    if up:
        iu = np.triu_indices(min(M, N))
        err = np.max(np.abs(C[iu] - ref[iu]))
        fl = 2.0 * K * (M * (M + 1) / 2)
    else:
        err = np.max(np.abs(C - ref))
        fl = 2.0 * M * N * K
    tf = fl / (ms.value * 1e-3) / 1e12 if ms.value > 0 else 0.0
    print(f"v{var} M={M} N={N} K={K} tA={tA} upper={up}: max err {err:.2e}  {ms.value*1e3:.1f} us  {tf:.2f} TF/s "
          f"({100*tf/37.1:.0f}% of DMMA peak)", flush=True)
    return err


if len(sys.argv) > 1 and sys.argv[1] == "--ncu":  # one launch per variant (ncu capture)
    for var in ([int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(20)):
        run(861, 861, 861, 0, 0, var=var, reps=0)
        run(861, 861, 861, 1, 1, var=var, reps=0)
    sys.exit(0)
for var in [7, 15, 16, 17, 18, 19]:
    for args in [(861, 861, 861, 0, 0), (861, 861, 861, 1, 1), (231, 231, 231, 0, 0)]:
        e = run(*args, var=var)
        assert e < 1e-11, (var, args)
for args in [(64, 64, 16, 0, 0), (100, 37, 53, 1, 0), (861, 861, 861, 0, 0), (861, 861, 861, 1, 0),
             (861, 861, 861, 1, 1), (231, 231, 231, 0, 0), (325, 325, 325, 1, 1), (1280, 1280, 1280, 0, 0),
             (861, 1722, 861, 1, 0), (7, 9, 1, 1, 0)]:
    e = run(*args)
    assert e < 1e-11, args
try:
    import torch
    a = torch.randn(861, 861, dtype=torch.float64, device="cuda")
    b = torch.randn(861, 861, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"cuBLAS (torch) 861^3 FP64: {ms*1e3:.1f} us {2*861**3/(ms*1e-3)/1e12:.2f} TF/s")
except Exception as ex:  # context only
    print("cuBLAS context skipped:", ex)
