"""GPU tests of the warm-started large-block PSD projection (csrc/warm.cuh; SURVEY §8(f) f4 "warm-started
... eig; iterates identical"; PAPER.md P:397-398 `eq:HsdeStep2`).

Unit level (sosadmm_debug_warm_project): a block a0 is projected by the cold eigensolver (seeding the
eigenvectors), then a perturbed a1 through the warm refinement; both projections are compared with the
plain LAPACK definition Pi_{S+}(a) = Q max(Lambda, 0) Q^T, and the refinement is checked to have been the
path that ran (status 1) whenever the perturbation is small.  Spectra with exact multiplicities, near-
degenerate clusters, eigenvalues crossing zero and a low-rank (SOS-like) PSD part exercise the cluster
solve; a large perturbation must fall back to the cold path and still be exact.

Solver level: a warm and a cold context (SOSADMM_WARM=0) iterate the same program; the iterates agree to
rounding, and the warm counters show the refinement carried the iterations."""
import ctypes
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = ctypes.POINTER(ctypes.c_double)


def lib():
    from paper_1708_04174_b200 import load_library

    L = load_library()
    L.sosadmm_debug_warm_project.argtypes = [ctypes.c_int, P, P, P, P, ctypes.POINTER(ctypes.c_int)]
    return L


def proj(a):
    lam, Q = np.linalg.eigh(a)
    return (Q * np.maximum(lam, 0.0)) @ Q.T


def warm_project(a0, a1):
    N = a0.shape[0]
    a0 = np.asfortranarray(a0)
    a1 = np.asfortranarray(a1)
    o0 = np.zeros((N, N), order="F")
    o1 = np.zeros((N, N), order="F")
    st = (ctypes.c_int * 6)()
    rc = lib().sosadmm_debug_warm_project(N, a0.ctypes.data_as(P), a1.ctypes.data_as(P), o0.ctypes.data_as(P),
                                          o1.ctypes.data_as(P), st)
    assert rc == 0
    return o0, o1, list(st)


def sym(rng, N):
    g = rng.standard_normal((N, N))
    return (g + g.T) / 2


def spectrum_matrix(rng, lam):
    Q, _ = np.linalg.qr(rng.standard_normal((len(lam), len(lam))))
    return (Q * lam) @ Q.T


def check(a0, a1, expect_warm):
    o0, o1, st = warm_project(a0, a1)
    for a, o in ((a0, o0), (a1, o1)):
        err = np.linalg.norm(o - proj(a)) / np.linalg.norm(a)
        assert err <= 1e-12, (err, st)
    if expect_warm:
        assert st[0] == 1, st  # the refinement, not the cold fallback, produced the projection
    return st


@pytest.mark.parametrize("N", [65, 231, 400, 861])
@pytest.mark.parametrize("delta", [0.0, 1e-8, 1e-5, 1e-3])
def test_warm_random_perturbation(N, delta):
    rng = np.random.default_rng(N)
    a0 = sym(rng, N)
    a1 = a0 + delta * sym(rng, N)
    st = check(a0, a1, expect_warm=True)
    if delta == 0.0:
        assert st[1] == 1, st  # an already-diagonalising basis certifies at the first evaluation


def test_warm_exact_multiplicities_and_clusters():
    rng = np.random.default_rng(7)
    N = 300
    lam = np.concatenate([np.full(40, 2.0), np.full(30, -1.5), 1.0 + 1e-11 * rng.standard_normal(20),
                          rng.standard_normal(N - 90)])
    a0 = spectrum_matrix(rng, lam)
    a1 = a0 + 1e-6 * sym(rng, N)
    st = check(a0, a1, expect_warm=True)
    assert st[5] >= 1, st


def test_warm_eigenvalue_crossing_zero():
    rng = np.random.default_rng(3)
    N = 200
    lam = np.concatenate([[1e-9, -2e-9, 5e-10], rng.standard_normal(N - 3)])
    Q, _ = np.linalg.qr(rng.standard_normal((N, N)))
    a0 = (Q * lam) @ Q.T
    lam1 = lam.copy()
    lam1[:3] = -lam1[:3]  # the three near-zero eigenvalues change sign
    a1 = (Q * lam1) @ Q.T + 1e-9 * sym(rng, N)
    check(a0, a1, expect_warm=False)  # either path: the result must be exact


def test_warm_low_rank_sos_like():
    """The SOS-program shape: a few positive eigenvalues (the Gram matrix's rank) and a large negative
    side, slowly changing (the ADMM iterate of a planted POP)."""
    rng = np.random.default_rng(11)
    N = 861
    lam = np.concatenate([np.abs(rng.standard_normal(16)) + 0.1, -np.abs(rng.standard_normal(N - 16)) - 1e-3])
    a0 = spectrum_matrix(rng, lam)
    a1 = a0 + 1e-5 * sym(rng, N) / np.sqrt(N)
    st = check(a0, a1, expect_warm=True)
    assert st[3] == 16 and st[4] == 0, st  # the positive side (16 columns) is the smaller one


def test_warm_large_change_falls_back():
    rng = np.random.default_rng(5)
    N = 150
    a0 = sym(rng, N)
    a1 = sym(rng, N)  # unrelated matrix: the refinement must give up, the cold path must still be exact
    st = check(a0, a1, expect_warm=False)
    assert st[0] == 2, st


def _iterates(warm, name, k):
    from paper_1708_04174_b200 import SosAdmm
    from sosgen import make_config

    old = os.environ.get("SOSADMM_WARM")
    os.environ["SOSADMM_WARM"] = "1" if warm else "0"
    try:
        g = SosAdmm.from_problem(make_config(name), tol=1e-300, max_iters=1 << 40)
    finally:
        if old is None:
            del os.environ["SOSADMM_WARM"]
        else:
            os.environ["SOSADMM_WARM"] = old
    g.iterate(k)
    it = g.get_iterate()
    ws = g.warm_stats()
    g.close()
    u = np.concatenate([it["xi"], it["y"], [it["tau"]], it["z"], it["s"], [it["kappa"]]])
    return u, ws


@pytest.mark.parametrize("name,k", [("pop20", 600), ("box24", 600)])
def test_warm_solver_matches_cold(name, k):
    uw, ws = _iterates(True, name, k)
    uc, wc = _iterates(False, name, k)
    assert ws[0]["enabled"] == 1 and wc[0]["enabled"] == 0
    assert ws[0]["warm"] >= k // 4, ws  # the refinement carried a large share of the iterations
    rel = np.linalg.norm(uw - uc) / np.linalg.norm(uc)
    assert rel <= 1e-9, rel  # BJ per-iterate parity tolerance; observed ~1e-12
