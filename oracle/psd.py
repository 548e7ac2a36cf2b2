"""PSD-cone projection in svec coordinates (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md P:281 defines S_+ as the (vectorised) PSD cone and P:397-398 projects onto it in
step `eq:HsdeStep2`.  svec is the isometry of S^N used on both sides (reading C1):
'U' packed column-major, position p(i, j) = i + j(j+1)/2 (i <= j), off-diagonals times sqrt(2).
The Euclidean projection of a symmetric matrix onto S_+ keeps the eigenvectors and clamps
negative eigenvalues to 0.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

_RT2 = np.sqrt(2.0)


def _pairs(N: int):
    jj = np.repeat(np.arange(N), np.arange(1, N + 1))
    ii = np.arange(N * (N + 1) // 2) - jj * (jj + 1) // 2
    return ii, jj


def smat(v: np.ndarray, N: int) -> np.ndarray:
    """svec^{-1}: symmetric N x N matrix of an svec vector."""
    ii, jj = _pairs(N)
    X = np.zeros((N, N))
    vals = np.where(ii == jj, v, v / _RT2)
    X[ii, jj] = vals
    X[jj, ii] = vals
    return X


def svec(X: np.ndarray) -> np.ndarray:
    N = X.shape[0]
    ii, jj = _pairs(N)
    return np.where(ii == jj, X[ii, jj], X[ii, jj] * _RT2)


def proj_psd(X: np.ndarray) -> np.ndarray:
    """Pi_{S+}(X) = Q diag(max(lambda, 0)) Q^T via LAPACK dsyevd (scipy driver 'evd')."""
    lam, Q = sla.eigh(X, driver="evd")
    Xp = (Q * np.maximum(lam, 0.0)) @ Q.T
    return 0.5 * (Xp + Xp.T)


def proj_psd_svec(v: np.ndarray, N: int) -> np.ndarray:
    return svec(proj_psd(smat(v, N)))
