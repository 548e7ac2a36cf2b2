"""GPU unit tests of the large-block PSD-projection stages (include/sosadmm_debug.h) against plain
numpy / LAPACK definitions: the DMMA GEMM, the cluster Householder tridiagonalisation (checked
through the similarity H T H^T = A it defines) and the divide-and-conquer tridiagonal
eigensolver (eigenvalues vs LAPACK, residual and orthogonality of the eigenvectors)."""
import ctypes

import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu

P = ctypes.POINTER(ctypes.c_double)


def lib():
    from paper_1708_04174_b200 import load_library

    L = load_library()
    L.sosadmm_debug_gemm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P]
    L.sosadmm_debug_tridiag.argtypes = [ctypes.c_int, P, P, P, P, P]
    L.sosadmm_debug_stedc.argtypes = [ctypes.c_int, P, P, P, P]
    L.sosadmm_debug_spdinv.argtypes = [ctypes.c_int, P]
    I = ctypes.POINTER(ctypes.c_int)
    L.sosadmm_debug_sy2sb.argtypes = [ctypes.c_int, P, P, P, P, I, I]
    L.sosadmm_debug_sb2st.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, P, P, I]
    L.sosadmm_debug_bt2.argtypes = [ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int, P]
    L.sosadmm_debug_tridiag2.argtypes = [ctypes.c_int, P, P, P, ctypes.POINTER(ctypes.c_float)]
    return L


def dp(a):
    return a.ctypes.data_as(P)


@pytest.mark.parametrize("M,N,K,tb", [(64, 64, 16, 0), (100, 37, 53, 0), (861, 861, 40, 1), (7, 130, 300, 1),
                                     (300, 257, 129, 0), (861, 700, 700, 0), (1280, 1100, 33, 1), (192, 192, 1, 0),
                                      (300, 5, 1, 0), (33, 33, 0, 0)])
def test_dmma_gemm(M, N, K, tb):
    rng = np.random.default_rng(M + N + K)
    A = np.asfortranarray(rng.standard_normal((M, K)))
    B = np.asfortranarray(rng.standard_normal((N, K) if tb else (K, N)))
    C = np.zeros((M, N), order="F")
    assert lib().sosadmm_debug_gemm(M, N, K, dp(A), dp(B), tb, dp(C)) == 0
    ref = A @ (B.T if tb else B)
    if K == 0:
        assert not C.any()
        return
    assert np.max(np.abs(C - ref)) <= 1e-14 * max(1, K) * (np.abs(A).max() * np.abs(B).max())


def _householder_Q(V, tau, N):
    Q = np.eye(N)
    for k in range(N - 2):
        v = V[:, k].copy()
        v[:k + 1] = 0.0
        Q = Q @ (np.eye(N) - tau[k] * np.outer(v, v))
    return Q


@pytest.mark.parametrize("N", [65, 100, 231, 285, 325, 513, 861, 1024, 1280])
def test_tridiag(N):
    rng = np.random.default_rng(N)
    G = rng.standard_normal((N, N))
    A = np.asfortranarray(G + G.T)
    d, e, tau = np.zeros(N), np.zeros(N - 1), np.zeros(N - 1)
    V = np.zeros((N, N), order="F")
    assert lib().sosadmm_debug_tridiag(N, dp(A), dp(d), dp(e), dp(tau), dp(V)) == 0
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    lam_T = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    lam_A = np.linalg.eigvalsh(A)
    assert np.max(np.abs(lam_T - lam_A)) <= 1e-12 * np.abs(lam_A).max() * np.sqrt(N)
    if N <= 325:
        Q = _householder_Q(V, tau, N)
        assert np.linalg.norm(Q @ T @ Q.T - A) <= 1e-13 * np.linalg.norm(A) * np.sqrt(N)


def _stedc(d, e):
    N = len(d)
    lam = np.zeros(N)
    Z = np.zeros((N, N), order="F")
    assert lib().sosadmm_debug_stedc(N, dp(np.ascontiguousarray(d)), dp(np.ascontiguousarray(e)), dp(lam), dp(Z)) == 0
    return lam, Z


@pytest.mark.parametrize("N,kind", [(2, "rand"), (3, "rand"), (17, "rand"), (65, "rand"), (231, "rand"),
                                    (861, "rand"), (300, "glued"), (200, "zero_e"), (129, "equal_d"),
                                    (500, "wilkinson"), (861, "clustered"), (1280, "rand"), (1024, "clustered"),
                                    # bottom nodes (k_dc_qrnode, n <= 16): one node, a few, graded, all zero
                                    (16, "rand"), (5, "wilkinson"), (33, "graded"), (48, "zero_all"),
                                    (40, "equal_d")])
def test_stedc(N, kind):
    rng = np.random.default_rng(N + len(kind))
    if kind == "rand":
        d, e = rng.standard_normal(N), rng.standard_normal(N - 1)
    elif kind == "glued":  # nearly decoupled blocks: tiny couplings
        d, e = rng.standard_normal(N), rng.standard_normal(N - 1)
        e[::25] = 1e-14
    elif kind == "zero_e":
        d, e = rng.standard_normal(N), rng.standard_normal(N - 1)
        e[::7] = 0.0
    elif kind == "equal_d":
        d, e = np.ones(N), 1e-3 * rng.standard_normal(N - 1)
    elif kind == "graded":  # eigenvalues over 16 orders of magnitude
        d = 10.0 ** (-16.0 * np.arange(N) / N)
        e = 1e-3 * np.sqrt(d[:-1] * d[1:]) * rng.standard_normal(N - 1)
    elif kind == "zero_all":
        d, e = np.zeros(N), np.zeros(N - 1)
    elif kind == "wilkinson":
        m = (N - 1) / 2
        d, e = np.abs(np.arange(N) - m), np.ones(N - 1)
    else:  # a low-rank-plus-noise spectrum tridiagonalised (many eigenvalues near 0)
        G = rng.standard_normal((N, 5))
        X = G @ G.T + 1e-12 * np.diag(rng.standard_normal(N))
        Tm = sla.hessenberg(X)
        d, e = np.diag(Tm).copy(), np.diag(Tm, 1).copy()
    lam, Z = _stedc(d, e)
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    ref = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    nrm = max(np.abs(ref).max(), 1e-300)
    assert np.all(np.diff(lam) >= 0)
    assert np.max(np.abs(lam - ref)) <= 1e-13 * nrm * np.sqrt(N)
    assert np.linalg.norm(T @ Z - Z * lam) <= 1e-13 * nrm * N
    assert np.linalg.norm(Z.T @ Z - np.eye(N)) <= 1e-13 * N


@pytest.mark.parametrize("t", [65, 130, 300, 1000, 2001])
def test_spd_inverse(t):
    rng = np.random.default_rng(t)
    G = rng.standard_normal((t, 3 * t // 2)) / np.sqrt(t)
    K = np.asfortranarray(np.eye(t) + G @ G.T)
    X = K.copy(order="F")
    assert lib().sosadmm_debug_spdinv(t, dp(X)) == 0
    assert np.linalg.norm(X @ K - np.eye(t)) <= 1e-12 * np.sqrt(t) * np.linalg.cond(K)


# ---------------------------------------------------------------------------------------------
# Two-stage tridiagonalisation (sy2sb.cuh dense -> band, sb2st.cuh band -> tridiagonal, bt2.cuh), each
# stage checked against the similarity it defines (the reflectors it returns, applied in numpy).

def _band_full(band, N, BW):
    """symmetric N x N matrix from the band layout band[c * 2BW + (r - c)], 0 <= r - c <= BW."""
    B = np.zeros((N, N))
    Bb = band.reshape(N, 2 * BW)
    for off in range(BW + 1):
        idx = np.arange(N - off)
        B[idx + off, idx] = Bb[idx, off]
    return np.tril(B) + np.tril(B, -1).T


def _sy2sb(A):
    N = A.shape[0]
    band = np.zeros(N * 32)
    V1 = np.zeros((N, N), order="F")
    tau1 = np.zeros(N)
    bw, nref = ctypes.c_int(0), ctypes.c_int(0)
    assert lib().sosadmm_debug_sy2sb(N, dp(np.asfortranarray(A)), dp(band), dp(V1), dp(tau1), ctypes.byref(bw),
                                     ctypes.byref(nref)) == 0
    return band[:N * 2 * bw.value], V1, tau1, bw.value, nref.value


@pytest.mark.parametrize("N", [65, 100, 231, 285, 325, 861, 946, 1280])
def test_sy2sb(N):
    rng = np.random.default_rng(N + 7)
    G = rng.standard_normal((N, N))
    A = G + G.T
    band, V1, tau1, BW, nref = _sy2sb(A)
    assert BW == (16 if N <= 880 else 8)
    B = _band_full(band, N, BW)
    lam_A = np.linalg.eigvalsh(A)
    assert np.max(np.abs(np.linalg.eigvalsh(B) - lam_A)) <= 1e-12 * np.abs(lam_A).max() * np.sqrt(N)
    if N <= 325:  # Q1 B Q1^T = A with Q1 = H_0 H_1 ... (H_k = I - tau_k v_k v_k^T, v_k = V1[k+1:, k])
        Q = np.eye(N)
        for k in range(nref):
            v = V1[:, k].copy()
            v[:k + 1] = 0.0
            assert np.all(v[k + 1:k + BW] == 0.0) and (tau1[k] == 0.0 or v[k + BW] == 1.0)
            Q = Q - tau1[k] * np.outer(Q @ v, v)
        assert np.linalg.norm(Q @ B @ Q.T - A) <= 1e-13 * np.linalg.norm(A) * np.sqrt(N)
        assert np.linalg.norm(Q.T @ Q - np.eye(N)) <= 1e-13 * np.sqrt(N)


def _random_band(N, BW, rng):
    band = np.zeros(N * 2 * BW)
    Bb = band.reshape(N, 2 * BW)
    for off in range(BW + 1):
        Bb[:N - off, off] = rng.standard_normal(N - off)
    return band


def _q2(V2, tau2, N, BW, KM):
    Q = np.eye(N)
    for i in range(N - 2):
        nt = (N - 2 - i) // BW + 1
        for k in range(nt):
            r0 = i + 1 + k * BW
            L = min(BW, N - r0)
            v = V2[(i * KM + k) * BW:(i * KM + k) * BW + L]
            Q[:, r0:r0 + L] -= tau2[i * KM + k] * np.outer(Q[:, r0:r0 + L] @ v, v)
    return Q


@pytest.mark.parametrize("N,BW", [(65, 16), (66, 16), (231, 16), (325, 16), (861, 16), (946, 8), (1280, 8)])
def test_sb2st(N, BW):
    rng = np.random.default_rng(N * 3 + BW)
    band = _random_band(N, BW, rng)
    B = _band_full(band, N, BW)
    KM = (N - 2) // BW + 1
    d, e = np.zeros(N), np.zeros(N - 1)
    V2, tau2 = np.zeros(N * KM * BW), np.zeros(N * KM)
    km = ctypes.c_int(0)
    assert lib().sosadmm_debug_sb2st(N, BW, dp(band), dp(d), dp(e), dp(V2), dp(tau2), ctypes.byref(km)) == 0
    assert km.value == KM
    lam_B = np.linalg.eigvalsh(B)
    lam_T = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    assert np.max(np.abs(lam_T - lam_B)) <= 1e-12 * np.abs(lam_B).max() * np.sqrt(N)
    if N <= 325:
        Q = _q2(V2, tau2, N, BW, KM)
        T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        assert np.linalg.norm(Q @ T @ Q.T - B) <= 1e-13 * np.linalg.norm(B) * np.sqrt(N)
    # the GPU back-transform of r columns applies the same Q2
    if N <= 325:
        r = min(N, 37)
        Z = np.asfortranarray(rng.standard_normal((N, r)))
        ref = Q @ Z
        assert lib().sosadmm_debug_bt2(N, BW, dp(V2), dp(tau2), r, dp(Z)) == 0
        assert np.max(np.abs(Z - ref)) <= 1e-13 * np.abs(ref).max() * np.sqrt(N)


@pytest.mark.parametrize("N", [65, 231, 285, 325, 861, 1280])
def test_tridiag_two_stage(N):
    rng = np.random.default_rng(N + 11)
    G = rng.standard_normal((N, N))
    A = np.asfortranarray(G + G.T)
    d, e = np.zeros(N), np.zeros(N - 1)
    ms = ctypes.c_float(0)
    assert lib().sosadmm_debug_tridiag2(N, dp(A), dp(d), dp(e), ctypes.byref(ms)) == 0
    lam_T = sla.eigh_tridiagonal(d, e, eigvals_only=True)
    lam_A = np.linalg.eigvalsh(A)
    assert np.max(np.abs(lam_T - lam_A)) <= 1e-12 * np.abs(lam_A).max() * np.sqrt(N)


@pytest.mark.parametrize("M,N,K,tA,up", [(861, 861, 861, 0, 0), (861, 861, 861, 1, 1), (231, 231, 231, 1, 0),
                                         (65, 33, 7, 0, 0), (100, 37, 53, 1, 0), (1280, 1280, 1280, 1, 1),
                                         (300, 5, 1, 0, 0), (7, 9, 1, 1, 0), (129, 129, 2, 1, 1)])
@pytest.mark.parametrize("variant", [-1, 0, 7])
def test_warm_dgemm(M, N, K, tA, up, variant):
    """The warm path's DMMA GEMM (dgemm.cuh) against numpy: op(A) = A or A^T, odd sizes (the 16-byte
    copies' zero-filled tails), upper-tile mode (only the tiles meeting the upper triangle are formed)."""
    L = lib()
    L.sosadmm_debug_dgemm.argtypes = [ctypes.c_int] * 3 + [P, ctypes.c_int, ctypes.c_int, P, P, ctypes.c_int,
                                                           ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    rng = np.random.default_rng(M * 7 + N * 3 + K + tA)
    A = np.asfortranarray(rng.standard_normal((K, M) if tA else (M, K)))
    B = np.asfortranarray(rng.standard_normal((K, N)))
    C = np.zeros((M, N), order="F")
    ms = ctypes.c_float(0)
    assert L.sosadmm_debug_dgemm(M, N, K, dp(A), tA, up, dp(B), dp(C), variant, 0, ctypes.byref(ms)) == 0
    ref = (A.T if tA else A) @ B
    tol = 1e-14 * max(1, K) * np.abs(A).max() * np.abs(B).max()
    if up:
        iu = np.triu_indices(min(M, N))
        assert np.max(np.abs(C[iu] - ref[iu])) <= tol
    else:
        assert np.max(np.abs(C - ref)) <= tol
