"""Oracle pins: residuals, termination classes and the refined linear step (readings C9, C15).

The paper fixes the outcome of the HSDE ("optimal solutions ... or a certificate of primal
or dual infeasibility ... from a nonzero solution"); SPEC S:329 / S:348 / S:364 give the residual
formulas that reading C9 adopts.  Each test evaluates the oracle at a point whose residuals are known
in closed form from the problem's construction (the planted KKT point of `sosgen.planted_kkt`, exact by
construction; a recession direction of an unbounded program), so a dropped /tau, swapped normalisers
or a wrong classification branch fails here, not only "GPU == oracle"."""
import numpy as np
import pytest

from oracle import HsdeOracle, OracleState, Status
from sosgen import make_config, planted_kkt, unbounded_pop
from sosgen.configs import svec


def _oracle(prob, b=None, c=None, refine=2):
    return HsdeOracle(prob.A, prob.b if b is None else b, prob.c if c is None else c, prob.n_free,
                      prob.psd_dims, refine=refine)


@pytest.mark.parametrize("name", ["pop6", "box24"])
@pytest.mark.parametrize("tau", [1.0, 0.3, 4.0])
def test_residuals_scale_free_at_kkt(name, tau):
    """The HSDE is a cone: (tau xi*, tau y*, tau, tau z*, 0, 0) is a solution for every tau > 0, and the
    scaled residuals (xi/tau, y/tau, z/tau) are those of the KKT point: ~0, pobj = -gamma0.  Dropping the
    /tau would give pres ~ |1 - tau| |b| / (1 + |b|) ~ 0.7."""
    prob = make_config(name)
    o = _oracle(prob)
    xi, y, z = planted_kkt(prob)
    st = OracleState(tau * xi, tau * y, tau, tau * z, np.zeros(prob.m), 0.0)
    r = o.residuals(st)
    assert r.pres < 1e-13 and r.dres < 1e-13 and r.gap < 1e-11, (r.pres, r.dres, r.gap)
    assert abs(r.pobj + prob.meta["gamma0"]) < 1e-12 and abs(r.dobj + prob.meta["gamma0"]) < 1e-11
    assert o.classify(r, 1e-6) == Status.OPTIMAL


@pytest.mark.parametrize("tau", [1.0, 0.3])
def test_primal_residual_normaliser(tau):
    """b perturbed by delta at an optimal point gives pres = |delta| / (1 + |b + delta|)
    (the problem solved is A xi = b + delta; the planted xi* meets A xi* = b exactly)."""
    prob = make_config("pop6")
    rng = np.random.default_rng(11)
    delta = rng.standard_normal(prob.m) * 1e-3
    bp = prob.b + delta
    o = _oracle(prob, b=bp)
    xi, y, z = planted_kkt(prob)
    r = o.residuals(OracleState(tau * xi, tau * y, tau, tau * z, np.zeros(prob.m), 0.0))
    want = np.linalg.norm(delta) / (1.0 + np.linalg.norm(bp))
    assert abs(r.pres - want) <= 1e-9 * want, (r.pres, want)
    assert r.dres < 1e-13
    # gap: c^T xi* = b^T y* = -gamma0, so with b + delta the dual objective moves by delta^T y*
    g0 = prob.meta["gamma0"]
    dob = -g0 + delta @ y
    gap = abs(-g0 - dob) / (1.0 + g0 + abs(dob))
    assert abs(r.gap - gap) <= 1e-9 * gap and abs(r.dobj - dob) <= 1e-11


@pytest.mark.parametrize("tau", [1.0, 0.3])
def test_dual_residual_normaliser(tau):
    """c perturbed by delta (on every column, PSD ones included) at the KKT point:
    dres = |A^T y + z - (c + delta)| / (1 + |c + delta|) = |delta| / (1 + |c + delta|)."""
    prob = make_config("box24")
    rng = np.random.default_rng(12)
    delta = rng.standard_normal(prob.n) * 1e-3
    cp = prob.c + delta
    o = _oracle(prob, c=cp)
    xi, y, z = planted_kkt(prob)
    r = o.residuals(OracleState(tau * xi, tau * y, tau, tau * z, np.zeros(prob.m), 0.0))
    want = np.linalg.norm(delta) / (1.0 + np.linalg.norm(cp))
    assert abs(r.dres - want) <= 1e-9 * want, (r.dres, want)
    assert r.pres < 1e-13
    assert abs(r.pobj - cp @ xi) <= 1e-11


def test_tau_zero_residuals_infinite():
    """tau = 0 gives infinite scaled residuals (no optimality claim from a zero tau)."""
    prob = make_config("pop6")
    o = _oracle(prob)
    xi, y, z = planted_kkt(prob)
    r = o.residuals(OracleState(xi, y, 0.0, z, np.zeros(prob.m), 1.0))
    assert r.pres == np.inf and r.dres == np.inf and r.gap == np.inf
    assert o.classify(r, 1e-4) != Status.OPTIMAL


def _gram_of_recession(nvars):
    """G with v2(x)^T G v2(x) = (1 + |x|^2)^2 (diagonal in the basis [1, x_i, x_i x_j])."""
    from sosgen.configs import basis

    B2 = basis(nvars, 0, 2)
    G = np.zeros((B2.shape[0], B2.shape[0]))
    for k, e in enumerate(B2):
        d = e.sum()
        if d == 0:
            G[k, k] = 1.0
        elif d == 1:
            G[k, k] = 2.0                       # 2 x_i^2
        elif e.max() == 2:
            G[k, k] = 1.0                       # x_i^4
        else:
            G[k, k] = 2.0                       # 2 x_i^2 x_j^2
    return G


@pytest.mark.parametrize("nvars", [1, 3])
def test_dual_infeasible_certificate_exact(nvars):
    """The recession direction (u = 1, X = G) of the unbounded program is a dual-infeasibility
    certificate: A xi = 0, xi in K, c^T xi = -1, so dinf = |A xi| / (-c^T xi) = 0 and the
    oracle's rule classifies it DUAL_INFEASIBLE (tau = 0, kappa > 0: P:361)."""
    prob = unbounded_pop(f"unb{nvars}", nvars)
    o = _oracle(prob)
    xi = np.concatenate([[1.0], svec(_gram_of_recession(nvars))])
    assert np.linalg.norm(prob.A @ xi) <= 1e-14 * np.linalg.norm(xi)
    st = OracleState(xi, np.zeros(prob.m), 0.0, np.zeros(prob.n), np.zeros(prob.m), 1.0)
    r = o.residuals(st)
    assert r.dinf <= 1e-14 and r.pinf == np.inf
    assert o.classify(r, 1e-4) == Status.DUAL_INFEASIBLE
    # the same xi with its sign flipped is not a certificate (c^T xi > 0)
    r2 = o.residuals(OracleState(-xi, np.zeros(prob.m), 0.0, np.zeros(prob.n), np.zeros(prob.m), 1.0))
    assert r2.dinf == np.inf and o.classify(r2, 1e-4) == Status.RUNNING


@pytest.mark.parametrize("nvars", [2, 6])
def test_dual_infeasible_solve(nvars):
    """HSDE-ADMM on the unbounded program ends DUAL_INFEASIBLE with a valid certificate: xi in K,
    c^T xi < 0, |A xi| <= tol (-c^T xi), tau = 0 < kappa."""
    prob = unbounded_pop(f"unb{nvars}", nvars)
    o = _oracle(prob)
    st, status, _ = o.solve(tol=1e-4, max_iters=5000)
    assert status == Status.DUAL_INFEASIBLE
    cx = o.c @ st.xi
    assert cx < 0 and np.linalg.norm(o.A @ st.xi) <= 1e-4 * (-cx)
    assert st.tau == 0.0 and st.kappa > 0.0
    N = prob.psd_dims[0]
    X = np.zeros((N, N))
    ii, jj = [], []
    for j in range(N):
        for i in range(j + 1):
            ii.append(i)
            jj.append(j)
    X[ii, jj] = st.xi[1:] / np.where(np.array(ii) == np.array(jj), 1.0, np.sqrt(2.0))
    X = X + np.triu(X, 1).T
    assert np.linalg.eigvalsh(X).min() >= -1e-12 * np.abs(X).max()


def test_classify_precedence():
    """C9: Optimal takes precedence over the certificate tests; PRIMAL before DUAL."""
    from oracle.hsde_admm import Residuals

    assert HsdeOracle.classify(Residuals(1e-5, 1e-5, 1e-5, 0, 0, 1e-6, 1e-6), 1e-4) == Status.OPTIMAL
    assert HsdeOracle.classify(Residuals(1.0, 1e-5, 1e-5, 0, 0, 1e-6, 1e-6), 1e-4) == Status.PRIMAL_INFEASIBLE
    assert HsdeOracle.classify(Residuals(1.0, 1e-5, 1e-5, 0, 0, 1.0, 1e-6), 1e-4) == Status.DUAL_INFEASIBLE
    assert HsdeOracle.classify(Residuals(1.0, 1e-5, 1e-5, 0, 0, 1.0, 1.0), 1e-4) == Status.RUNNING


def _affine_ld_diagonal(prob, w1, w2, w3):
    """(I + Q)^{-1} w in extended precision for programs where A A^T is diagonal (every column has at most
    one nonzero: configs 0, 1, 4), by eliminating u1 and u2 in the order of the equations of
    `eq:DefinitionQ` — an independent route from the oracle's KKT LU + refinement:
      (I + A A^T) u2 = w2 - A w1 + (b + A c) u3,   u1 = w1 - c u3 + A^T u2,   -c^T u1 + b^T u2 + u3 = w3."""
    LD = np.longdouble
    A = prob.A.tocsr().astype(LD)
    AT = prob.A.T.tocsr().astype(LD)
    b, c = prob.b.astype(LD), prob.c.astype(LD)
    Ad = prob.A.tocoo()
    dg = np.ones(prob.m, dtype=LD)
    np.add.at(dg, Ad.row, Ad.data.astype(LD) ** 2)
    w1, w2, w3 = w1.astype(LD), w2.astype(LD), LD(w3)
    p2 = (w2 - A @ w1) / dg
    q2 = (b + A @ c) / dg
    a0 = -(c @ (w1 + AT @ p2)) + b @ p2
    a1 = -(c @ (-c + AT @ q2)) + b @ q2 + 1
    u3 = (w3 - a0) / a1
    u2 = p2 + u3 * q2
    return w1 - c * u3 + AT @ u2, u2, u3


def test_refined_linear_step_long_double_pin():
    """Reading C15: the refined oracle solves the paper's linear system to working accuracy.  pop20, the
    first iteration's input omega = u0 + v0 = (0, 0, 1): u_hat_3 within 1e-14 relative of an
    extended-precision solve (the unrefined one-pass formula is ~4e-6 off, which this catches)."""
    prob = make_config("pop20")
    Ad = (prob.A @ prob.A.T).tocoo()
    assert not np.any(Ad.data[Ad.row != Ad.col])  # A A^T diagonal (Proposition 1 + A_1 = e_const)
    w1, w2, w3 = np.zeros(prob.n), np.zeros(prob.m), 1.0
    r1, r2, r3 = _affine_ld_diagonal(prob, w1, w2, w3)
    u1, u2, u3 = _oracle(prob).affine(w1, w2, w3)
    assert abs(u3 - float(r3)) <= 1e-14 * abs(float(r3))
    assert np.linalg.norm((u1 - r1).astype(float)) <= 1e-15 * np.linalg.norm(r1.astype(float))
    assert np.linalg.norm((u2 - r2).astype(float)) <= 1e-15 * np.linalg.norm(r2.astype(float))
    v1, v2, v3 = _oracle(prob, refine=0).affine(w1, w2, w3)
    assert abs(v3 - float(r3)) > 1e-10 * abs(float(r3))  # the pin has teeth


def test_refined_linear_step_general_state():
    """Same pin at a generic right-hand side (random omega) on pop6: all three blocks to 1e-14."""
    prob = make_config("pop6")
    rng = np.random.default_rng(5)
    w1, w2, w3 = rng.standard_normal(prob.n), rng.standard_normal(prob.m), 0.7
    r1, r2, r3 = _affine_ld_diagonal(prob, w1, w2, w3)
    u1, u2, u3 = _oracle(prob).affine(w1, w2, w3)
    assert abs(u3 - float(r3)) <= 1e-14 * max(abs(float(r3)), 1.0)
    assert np.linalg.norm((u1 - r1).astype(float)) <= 1e-14 * np.linalg.norm(r1.astype(float))
    assert np.linalg.norm((u2 - r2).astype(float)) <= 1e-14 * np.linalg.norm(r2.astype(float))
