"""Per-phase clock breakdown of the cluster tridiagonalisation (sosadmm_debug_tridiag_prof)."""
import ctypes
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1708_04174_b200 import load_library  # noqa: E402

P = ctypes.POINTER(ctypes.c_double)
L = load_library()
L.sosadmm_debug_tridiag_prof.argtypes = [ctypes.c_int, P, ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_float)]
for N in [int(x) for x in (sys.argv[1:] or ["861"])]:
    rng = np.random.default_rng(N)
    G = rng.standard_normal((N, N))
    A = np.asfortranarray(G + G.T)
    prof = np.zeros((N - 2) * 8, dtype=np.int64)
    ms = ctypes.c_float(0)
    rc = L.sosadmm_debug_tridiag_prof(N, A.ctypes.data_as(P), prof.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                      ctypes.byref(ms))
    assert rc == 0, rc
    pr = prof.reshape(N - 2, 8).astype(np.float64)
    step = np.diff(pr[:, 0])  # cycles per step
    names = ["A:reflector+setup", "X:fused pass", "X:col sums+push+rowsum", "blocksum(d)", "push sd/se + wait Q",
             "Y:w,x", "Y:blocksum+push", "wait Y"]
    d = np.zeros((N - 3, 8))
    for p in range(7):
        d[:, p] = pr[:-1, p + 1] - pr[:-1, p]
    d[:, 7] = pr[1:, 0] - pr[:-1, 7]
    print(f"N={N}: launch {ms.value:.3f} ms, {ms.value * 1e3 / (N - 2):.2f} us/step, mean {step.mean():.0f} cycles/step")
    for lo, hi in [(0, 50), (N // 3, N // 3 + 50), (2 * N // 3, 2 * N // 3 + 50), (N - 60, N - 10)]:
        print(f"  k in [{lo},{hi}):", " ".join(f"{names[p]}={d[lo:hi, p].mean():.0f}" for p in range(8)))
