"""Time the two-stage tridiagonalisation (sosadmm_debug_tridiag2) against the one-cluster kernel."""
import ctypes
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1708_04174_b200 import load_library

P = ctypes.POINTER(ctypes.c_double)
L = load_library()
L.sosadmm_debug_tridiag2.argtypes = [ctypes.c_int, P, P, P, ctypes.POINTER(ctypes.c_float)]
L.sosadmm_debug_tridiag_prof.argtypes = [ctypes.c_int, P, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_float)]
dp = lambda a: a.ctypes.data_as(P)
for N in [int(x) for x in (sys.argv[1:] or ["66", "231", "285", "325", "861", "946", "1280"])]:
    rng = np.random.default_rng(N)
    G = rng.standard_normal((N, N))
    A = np.asfortranarray(G + G.T)
    d, e = np.zeros(N), np.zeros(N - 1)
    ts = []
    for _ in range(3):
        ms = ctypes.c_float(0)
        rc = L.sosadmm_debug_tridiag2(N, dp(A), dp(d), dp(e), ctypes.byref(ms))
        ts.append(ms.value)
    prof = np.zeros(16 * N, dtype=np.int64)
    ms1 = ctypes.c_float(0)
    rc1 = L.sosadmm_debug_tridiag_prof(N, dp(A), prof.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), ctypes.byref(ms1))
    print(f"N={N} two-stage rc={rc} ms={min(ts):.3f} (runs {['%.3f' % t for t in ts]})  one-stage rc={rc1} ms={ms1.value:.3f}", flush=True)
