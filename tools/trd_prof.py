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
    prof = np.zeros((N - 2) * 16, dtype=np.int64)
    ms = ctypes.c_float(0)
    rc = L.sosadmm_debug_tridiag_prof(N, A.ctypes.data_as(P), prof.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)),
                                      ctypes.byref(ms))
    assert rc == 0, rc
    pr = prof.reshape(N - 2, 16).astype(np.float64)
    # stamp order within a step: 0, 1 (registers set up), 2, 3, 4, 8, 5, 10, 11, 7
    order = [0, 1, 2, 3, 4, 8, 5, 10, 11, 7]
    names = ["regs", "X:fused", "X:colsum+push+sync", "tid<C push", "prow", "wait Q",
             "Y:sums", "Y:rows+push", "V store", "wait Y"]
    n = N - 3
    d = np.zeros((n, len(order)))
    for p in range(len(order) - 1):
        d[:, p] = pr[:n, order[p + 1]] - pr[:n, order[p]]
    d[:, -1] = pr[1:n + 1, 0] - pr[:n, 7]
    step = np.diff(pr[:, 0])
    print(f"N={N}: launch {ms.value:.3f} ms, {ms.value * 1e3 / (N - 2):.2f} us/step, median {np.median(step):.0f} cycles/step")
    for lo, hi in [(0, 50), (N // 3, N // 3 + 50), (2 * N // 3, 2 * N // 3 + 50), (N - 60, N - 10)]:
        print(f"  k in [{lo},{hi}):", " ".join(f"{names[p]}={np.median(d[lo:hi, p]):.0f}" for p in range(len(order))))
        if False:
            sub = [np.median(pr[lo:hi, 13] - pr[lo:hi, 0]), np.median(pr[lo:hi, 14] - pr[lo:hi, 13]),
                   np.median(pr[lo:hi, 15] - pr[lo:hi, 14]), np.median(pr[lo:hi, 8] - pr[lo:hi, 15])]
            print("     warp0: top->start %.0f  sum+alpha %.0f  sqrt %.0f  divs %.0f" % tuple(sub))
