"""Oracle pins: PSD-cone projection."""
import numpy as np
import pytest

from oracle import proj_psd_svec, smat, svec
from oracle.psd import proj_psd


def test_diag_example():
    assert np.array_equal(proj_psd(np.diag([1.0, -2.0])), np.diag([1.0, 0.0]))


def test_svec_isometry():
    rng = np.random.default_rng(0)
    for N in [1, 2, 5, 13]:
        X = rng.standard_normal((N, N)); X = X + X.T
        Y = rng.standard_normal((N, N)); Y = Y + Y.T
        assert abs(svec(X) @ svec(Y) - np.trace(X @ Y)) < 1e-12 * (1 + np.abs(X).sum() * np.abs(Y).sum())
        assert np.allclose(smat(svec(X), N), X, rtol=0, atol=1e-15 * np.abs(X).max())


@pytest.mark.parametrize("N", [1, 3, 8, 28])
def test_projection_properties(N):
    rng = np.random.default_rng(N)
    L = N * (N + 1) // 2
    for _ in range(4):
        a = rng.standard_normal(L)
        b = rng.standard_normal(L)
        pa, pb = proj_psd_svec(a, N), proj_psd_svec(b, N)
        # in the cone
        assert np.linalg.eigvalsh(smat(pa, N)).min() >= -1e-13 * np.linalg.norm(a)
        # idempotent
        assert np.linalg.norm(proj_psd_svec(pa, N) - pa) <= 1e-13 * np.linalg.norm(a)
        # Moreau: a = P(a) - P(-a), <P(a), P(a) - a> = 0
        assert np.linalg.norm(pa - proj_psd_svec(-a, N) - a) <= 1e-13 * np.linalg.norm(a)
        assert abs(pa @ (pa - a)) <= 1e-12 * (a @ a)
        # nonexpansive
        assert np.linalg.norm(pa - pb) <= np.linalg.norm(a - b) + 1e-12


def test_psd_input_unchanged():
    rng = np.random.default_rng(3)
    G = rng.standard_normal((7, 4))
    X = G @ G.T
    assert np.linalg.norm(proj_psd(X) - X) <= 1e-13 * np.linalg.norm(X)
