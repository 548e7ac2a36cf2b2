"""Oracle pins: the linear step u_hat = (I + Q)^{-1} omega.

Pinned against the HSDE definition itself (Q materialised from A, b, c as printed at
P:377-379) and against a dense LU of I + Q — neither uses the oracle's KKT/SMW route."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import HsdeOracle
from sosgen import make_config, univariate_feasibility, ball_pop
from sosgen.configs import planted_pop


def Q_sparse(A, b, c):
    """Q of `eq:DefinitionQ`."""
    m, n = A.shape
    bc = sp.csc_matrix(c.reshape(-1, 1))
    bb = sp.csc_matrix(b.reshape(-1, 1))
    return sp.bmat([[None, -A.T, bc], [A, None, -bb], [-bc.T, bb.T, None]], format="csc")


def _omega(o, rng):
    return rng.standard_normal(o.n), rng.standard_normal(o.m), float(rng.standard_normal())


@pytest.mark.parametrize("maker", [lambda: make_config("pop6"), lambda: make_config("box24"),
                                   lambda: make_config("lyap10"), lambda: ball_pop(6)])
def test_round_trip_I_plus_Q(maker):
    prob = maker()
    o = HsdeOracle.from_problem(prob)
    Q = Q_sparse(o.A, o.b, o.c)
    rng = np.random.default_rng(1)
    for _ in range(3):
        w1, w2, w3 = _omega(o, rng)
        u1, u2, u3 = o.affine(w1, w2, w3)
        u = np.concatenate([u1, u2, [u3]])
        w = np.concatenate([w1, w2, [w3]])
        res = u + Q @ u - w
        # u_hat_3 = w3 + c^T u_hat_1 - b^T u_hat_2 cancels terms of size |b||u_hat_2|, and row 2
        # multiplies that rounding by |b| again (box24: |b| = 1.5e3).  A wrong sign, index or dropped
        # term gives an O(|w|) residual instead.
        canc = np.linalg.norm(o.b) * (abs(o.c) @ abs(u1) + abs(o.b) @ abs(u2))
        scale = np.linalg.norm(w) + np.linalg.norm(Q @ u) + canc
        assert np.linalg.norm(res) <= 1e-14 * scale
        assert np.linalg.norm(res) <= 1e-6 * np.linalg.norm(w)


def test_Q_skew_and_denominator():
    prob = make_config("pop6")
    o = HsdeOracle.from_problem(prob)
    Q = Q_sparse(o.A, o.b, o.c)
    assert abs(Q + Q.T).max() == 0.0
    # M + M^T = 2I  =>  zeta^T M^{-1} zeta = ||M^{-1} zeta||^2 >= 0, so denom >= 1
    assert o.denom >= 1.0
    assert abs((o.denom - 1.0) - o.h @ o.h) <= 1e-10 * (o.h @ o.h)


@pytest.mark.parametrize("maker", [lambda: univariate_feasibility("sq", [1.0, 2.0, 1.0]),
                                   lambda: planted_pop("p2", 2, 2, seed=3),
                                   lambda: ball_pop(2)])
def test_dense_lu_agrees(maker):
    """u_hat matches a dense LU solve of the materialised I + Q."""
    prob = maker()
    o = HsdeOracle.from_problem(prob)
    Qd = Q_sparse(o.A, o.b, o.c).toarray()
    I = np.eye(Qd.shape[0])
    rng = np.random.default_rng(7)
    for _ in range(3):
        w1, w2, w3 = _omega(o, rng)
        u_ref = np.linalg.solve(I + Qd, np.concatenate([w1, w2, [w3]]))
        u1, u2, u3 = o.affine(w1, w2, w3)
        u = np.concatenate([u1, u2, [u3]])
        assert np.linalg.norm(u - u_ref) <= 1e-12 * np.linalg.norm(u_ref)


def test_zero_in_zero_out():
    o = HsdeOracle.from_problem(make_config("pop6"))
    u1, u2, u3 = o.affine(np.zeros(o.n), np.zeros(o.m), 0.0)
    assert not u1.any() and not u2.any() and u3 == 0.0
