"""Debug / timing of the two-stage path: per-stage times, and the lowrank N=861 projection stages."""
import ctypes
import sys
import numpy as np
import scipy.linalg as sla
sys.path.insert(0, ".")
from paper_1708_04174_b200 import load_library
from oracle import proj_psd_svec, svec

P = ctypes.POINTER(ctypes.c_double)
F = ctypes.POINTER(ctypes.c_float)
I = ctypes.POINTER(ctypes.c_int)
L = load_library()
LL = ctypes.POINTER(ctypes.c_longlong)
L.sosadmm_debug_ts_timing.argtypes = [ctypes.c_int, P, F, F, LL, LL]
L.sosadmm_debug_psd_stages.argtypes = [ctypes.c_int, P, P, P, P, I]
dp = lambda a: a.ctypes.data_as(P)
for N in [int(x) for x in (sys.argv[1:] or ["66", "231", "325", "861", "1280"])]:
    rng = np.random.default_rng(N)
    G = rng.standard_normal((N, N))
    A = np.asfortranarray(G + G.T)
    m1, m2 = ctypes.c_float(0), ctypes.c_float(0)
    BW = 16 if N <= 880 else 8
    Pn = (N - 1) // BW
    p1 = np.zeros(16 * (Pn + 1), dtype=np.int64)
    p2 = np.zeros(4 * ((N - 2) // BW + 1), dtype=np.int64)
    rc = L.sosadmm_debug_ts_timing(N, dp(A), ctypes.byref(m1), ctypes.byref(m2), p1.ctypes.data_as(LL),
                                   p2.ctypes.data_as(LL))
    print(f"N={N} rc={rc} stage1 {m1.value:.3f} ms  stage2 {m2.value:.3f} ms", flush=True)
    pr = p1.reshape(-1, 16).astype(np.float64)
    if Pn > 2:
        # panel CTA: wait-panel, slice, QR, publish, wait-y, S, corr ; worker 0: wait-v, Y, wait-y, first, wait-s, bulk
        pc = np.diff(pr[1:Pn - 1, 0:8], axis=1).mean(axis=0)
        wk = np.diff(pr[1:Pn - 1, 8:15], axis=1).mean(axis=0)
        per = np.diff(pr[1:Pn - 1, 0]).mean()
        print(f"   cycles/panel {per:.0f}; panel CTA [wait_panel, slice, qr, publish, wait_y, S, -] "
              f"{np.round(pc).astype(int).tolist()}", flush=True)
        print(f"   worker0 [wait_v, Y, wait_y, wait_s, first+publish, bulk] {np.round(wk).astype(int).tolist()}",
              flush=True)
    nt0 = (N - 2) // BW + 1
    if nt0 > 3:
        st = p2[:4 * nt0].reshape(nt0, 4).astype(np.float64)
        per_task = np.diff(st[1:, 3]).mean()
        ph = np.array([st[2:, 0] - st[1:-1, 3], st[2:, 1] - st[2:, 0], st[2:, 2] - st[2:, 1], st[2:, 3] - st[2:, 2]]).mean(axis=1)
        print(f"   stage2 sweep-0 cycles/task {per_task:.0f}: [right, house, left, two-sided] {np.round(ph).astype(int).tolist()}",
              flush=True)
for N in [231, 861]:
    rng = np.random.default_rng(3)
    G = rng.standard_normal((N, 3)); H = rng.standard_normal((N, 2))
    X = np.asfortranarray(G @ G.T - H @ H.T + 1e-10 * np.eye(N))
    d, e, lam = np.zeros(N), np.zeros(N - 1), np.zeros(N)
    sel = np.zeros(3, dtype=np.int32)
    rc = L.sosadmm_debug_psd_stages(N, dp(X), dp(d), dp(e), dp(lam), sel.ctypes.data_as(I))
    ref = np.linalg.eigvalsh(X)
    lt = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    print(f"lowrank N={N} rc={rc} sel={sel.tolist()} |eig(T)-eig(X)|={np.abs(lt - ref).max():.3e} "
          f"|lam-eig(X)|={np.abs(np.sort(lam) - ref).max():.3e} neg={np.sum(ref < 0)} pos={np.sum(ref > 0)}", flush=True)
    print("   smallest:", ref[:4], " lam:", np.sort(lam)[:4])
