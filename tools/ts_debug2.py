"""Localise the two-stage failure on the low-rank N = 861 input: stage 1 determinism and similarity,
stage 2 eigenvalues."""
import ctypes
import sys
import numpy as np
import scipy.linalg as sla
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1708_04174_b200 import load_library
import test_gpu_stages as T

L = T.lib()
for N, kind in [(861, "lowrank"), (861, "gauss"), (500, "lowrank"), (325, "lowrank")]:
    rng = np.random.default_rng(3)
    if kind == "lowrank":
        G = rng.standard_normal((N, 3)); H = rng.standard_normal((N, 2))
        X = G @ G.T - H @ H.T + 1e-10 * np.eye(N)
    else:
        G = rng.standard_normal((N, N)); X = G + G.T
    b1, V1, tau1, BW, nref = T._sy2sb(X)
    b2, V1b, tau1b, _, _ = T._sy2sb(X)
    B1 = T._band_full(b1, N, BW)
    lamX = np.linalg.eigvalsh(X)
    print(f"N={N} {kind}: stage1 deterministic={np.array_equal(b1, b2) and np.array_equal(V1, V1b)} "
          f"|eig(B)-eig(X)|={np.abs(np.linalg.eigvalsh(B1) - lamX).max():.3e}", flush=True)
    Q = np.eye(N)
    for k in range(nref):
        v = V1[:, k].copy(); v[:k + 1] = 0.0
        Q = Q - tau1[k] * np.outer(Q @ v, v)
    Bref = Q.T @ X @ Q
    outside = np.abs(np.tril(Bref, -BW - 1)).max()
    diff = np.abs(np.tril(Bref) - np.tril(B1)).max()
    # first column where the band differs
    colerr = np.abs(np.tril(Bref) - np.tril(B1)).max(axis=0)
    bad = np.nonzero(colerr > 1e-9 * np.abs(X).max())[0]
    print(f"   Q1^T X Q1 outside band {outside:.3e}, band diff {diff:.3e}, first bad column {bad[:5]} of {len(bad)}",
          flush=True)
    KM = (N - 2) // BW + 1
    d, e = np.zeros(N), np.zeros(N - 1)
    V2, tau2 = np.zeros(N * KM * BW), np.zeros(N * KM)
    km = ctypes.c_int(0)
    L.sosadmm_debug_sb2st(N, BW, T.dp(b1), T.dp(d), T.dp(e), T.dp(V2), T.dp(tau2), ctypes.byref(km))
    lt = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    print(f"   stage2 |eig(T)-eig(B)|={np.abs(lt - np.linalg.eigvalsh(B1)).max():.3e}", flush=True)
