"""The five BASELINE.json configs, the tiny textbook programs, and planted KKT points.

Seeded input generation (readings C5, C6, C12).  Draw order per
instance (C12): numpy PCG64 `default_rng(seed)`; first x0, then C in R^{K x N} (row k = the
coefficients of q_k in the Gram basis order, the constant shift applied afterwards); for the
Lyapunov config, H in R^{n x 220}.

Planted POP (BASELINE.json configs 0, 1, 3, 4): p(x) = gamma0 + sum_k q_k(x)^2 with q_k(x0) = 0,
so p - gamma0 is SOS and p(x0) = gamma0: the optimum of max{gamma : p - gamma SOS} is gamma0
(PAPER.md `eq:POPsdp`).
"""
from __future__ import annotations

from math import comb

import numpy as np

from .monomials import basis_tuples, exponents
from .problem import GramBlock, Poly, Problem, SosConstraint, assemble, svec_pairs

SQRT2 = float(np.sqrt(2.0))

CONFIG_NAMES = ["pop6", "pop20", "lyap10", "box24", "pop40"]
DEFAULT_SEEDS = {"pop6": 0, "pop20": 0, "lyap10": 0, "box24": 0, "pop40": 0}


def basis(nvars: int, dmin: int, dmax: int) -> np.ndarray:
    return exponents(basis_tuples(nvars, dmin, dmax), nvars)


def _square_coeffs(C: np.ndarray, B: np.ndarray):
    """Exponents and coefficients of sum_k (C_k . v_B(x))^2 (duplicates not merged)."""
    N = B.shape[0]
    ii, jj = svec_pairs(N)
    ex = B[ii] + B[jj]
    w = np.where(ii == jj, 1.0, 2.0)
    coef = (C[:, ii] * C[:, jj]).sum(axis=0) * w
    return ex, coef


def planted_pop(name: str, nvars: int, K: int, seed: int, gamma0: float = 1.0, box: bool = False) -> Problem:
    """max gamma s.t. p - gamma SOS (unconstrained) or p - gamma = s0 + sum_i s_i (1 - x_i^2) (box)."""
    rng = np.random.default_rng(seed)
    if box:
        x0 = rng.uniform(-0.5, 0.5, size=nvars)
    else:
        x0 = rng.standard_normal(nvars)
    B2 = basis(nvars, 0, 2)
    N = B2.shape[0]
    C = rng.standard_normal((K, N))
    vx0 = np.prod(np.power(x0[None, :], B2), axis=1)
    C[:, 0] -= C @ vx0  # q_k(x0) = 0 (basis entry 0 is the constant monomial)
    ex, coef = _square_coeffs(C, B2)
    ex = np.concatenate([np.zeros((1, nvars), dtype=np.int64), ex])
    coef = np.concatenate([[gamma0], coef])
    p = Poly(coef, ex)
    one = Poly.const(nvars, 1.0)
    blocks = []
    if box:
        B1 = basis(nvars, 0, 1)
        for i in range(nvars):
            e2 = np.zeros((2, nvars), dtype=np.int64)
            e2[1, i] = 2
            blocks.append(GramBlock(B1, Poly(np.array([1.0, -1.0]), e2)))
    blocks.append(GramBlock(B2))
    con = SosConstraint(g0=p, g=[one], blocks=blocks)
    meta = dict(kind="box_pop" if box else "pop", nvars=nvars, K=K, seed=seed, gamma0=gamma0,
                x0=x0.tolist(), C=C.tolist())
    prob = assemble(name, nvars, [con], np.array([-1.0]), meta)
    return prob


def lyapunov(name: str, nvars: int, seed: int, eps: float = 1e-3, h_scale: float = 0.05,
             zero_h: bool = False) -> Problem:
    """BASELINE.json config 2 (PAPER.md `eq:Lyapunovsdp`; reading C6).

    f = -x + h(x), h_i = sum_{|nu|=3} H_{i nu} x^nu; V = sum_{1<=|mu|<=4} u_mu x^mu;
    s1 = V - eps |x|^2 (Gram basis deg 1..2), s2 = -grad V . f - eps |x|^2 (Gram basis deg 1..3).
    """
    rng = np.random.default_rng(seed)
    cub = basis(nvars, 3, 3)
    H = rng.normal(0.0, h_scale, size=(nvars, cub.shape[0]))
    if zero_h:
        H[:] = 0.0
    mus = basis(nvars, 1, 4)
    t = mus.shape[0]
    sq = np.zeros((nvars, nvars), dtype=np.int64)
    sq[np.arange(nvars), np.arange(nvars)] = 2
    g0 = Poly(np.full(nvars, -eps), sq)
    # constraint 1: s1 = g0 - sum u_mu g_mu with g_mu = -x^mu
    g1 = [Poly(np.array([-1.0]), mus[k:k + 1]) for k in range(t)]
    # constraint 2: g'_mu = grad(x^mu) . f = -|mu| x^mu + sum_i mu_i sum_nu H_{i nu} x^(mu - e_i + nu)
    g2 = []
    for k in range(t):
        mu = mus[k]
        ex = [mu[None, :]]
        co = [np.array([-float(mu.sum())])]
        for i in range(nvars):
            if mu[i] == 0:
                continue
            base = mu.copy()
            base[i] -= 1
            nz = H[i] != 0
            ex.append(base[None, :] + cub[nz])
            co.append(mu[i] * H[i][nz])
        ex = np.concatenate(ex)
        co = np.concatenate(co)
        # merge duplicate monomials
        e8 = np.ascontiguousarray(ex.astype(np.int8)).view(np.dtype((np.void, nvars))).ravel()
        u, inv = np.unique(e8, return_inverse=True)
        cm = np.zeros(len(u))
        np.add.at(cm, inv, co)
        first = np.zeros(len(u), dtype=np.int64)
        first[inv[::-1]] = np.arange(len(inv))[::-1]
        g2.append(Poly(cm, ex[first]))
    con1 = SosConstraint(g0=g0, g=g1, blocks=[GramBlock(basis(nvars, 1, 2))])
    con2 = SosConstraint(g0=g0, g=g2, blocks=[GramBlock(basis(nvars, 1, 3))])
    meta = dict(kind="lyapunov", nvars=nvars, seed=seed, eps=eps, h_scale=h_scale, zero_h=zero_h)
    return assemble(name, nvars, [con1, con2], np.zeros(t), meta)


def ball_pop(nvars: int) -> Problem:
    """PAPER.md `eq:ExamplePOP`: Lasserre order 2d = 4, weighted form (§VI) with
    p1 = 1 - sum x_i^2: p - gamma = s0 + s1 p1, s0 Gram over deg <= 2, s1 Gram over deg <= 1."""
    n = nvars
    terms_e, terms_c = [], []
    for i in range(n):
        for j in range(i + 1, n):
            for (a, bb, cc) in [((i, j), None, 1.0), ((i, i, j), None, 1.0), ((j, j, j), None, -1.0),
                                ((i, i, j, j), None, -1.0)]:
                e = np.zeros(n, dtype=np.int64)
                for v in a:
                    e[v] += 1
                terms_e.append(e)
                terms_c.append(cc)
    ex = np.array(terms_e)
    e8 = np.ascontiguousarray(ex.astype(np.int8)).view(np.dtype((np.void, n))).ravel()
    u, inv = np.unique(e8, return_inverse=True)
    cm = np.zeros(len(u))
    np.add.at(cm, inv, np.array(terms_c))
    first = np.zeros(len(u), dtype=np.int64)
    first[inv[::-1]] = np.arange(len(inv))[::-1]
    p = Poly(cm, ex[first])
    e2 = np.zeros((n + 1, n), dtype=np.int64)
    for i in range(n):
        e2[i + 1, i] = 2
    p1 = Poly(np.concatenate([[1.0], -np.ones(n)]), e2)
    con = SosConstraint(g0=p, g=[Poly.const(n, 1.0)],
                        blocks=[GramBlock(basis(n, 0, 1), p1), GramBlock(basis(n, 0, 2))])
    return assemble(f"ballpop{n}", n, [con], np.array([-1.0]), dict(kind="ball_pop", nvars=n))


def unbounded_pop(name: str, nvars: int) -> Problem:
    """A dual-infeasible (primal-unbounded) program for the DUAL_INFEASIBLE status (
    PAPER.md P:361 "certificate of ... dual infeasibility"): max u s.t. 1 + u (1 + |x|^2)^2 SOS over the
    Gram basis of degree <= 2.  (1 + |x|^2)^2 is SOS, so every u >= 0 is feasible and the objective -u is
    unbounded below.  Recession direction: u = 1, X = G with v2(x)^T G v2(x) = (1 + |x|^2)^2
    (A xi = 0, xi in K, c^T xi = -1 < 0).  No random draws."""
    # (1 + |x|^2)^2 = 1 + 2 sum_i x_i^2 + sum_i x_i^4 + 2 sum_{i<j} x_i^2 x_j^2
    ex, co = [np.zeros(nvars, dtype=np.int64)], [1.0]
    for i in range(nvars):
        e = np.zeros(nvars, dtype=np.int64)
        e[i] = 2
        ex.append(e)
        co.append(2.0)
        e4 = np.zeros(nvars, dtype=np.int64)
        e4[i] = 4
        ex.append(e4)
        co.append(1.0)
        for j in range(i + 1, nvars):
            eij = np.zeros(nvars, dtype=np.int64)
            eij[i] = eij[j] = 2
            ex.append(eij)
            co.append(2.0)
    g1 = Poly(-np.array(co), np.array(ex))
    con = SosConstraint(g0=Poly.const(nvars, 1.0), g=[g1], blocks=[GramBlock(basis(nvars, 0, 2))])
    return assemble(name, nvars, [con], np.array([-1.0]), dict(kind="unbounded_pop", nvars=nvars))


def edge_program(kind: str, seed: int = 0) -> Problem:
    """Degenerate conic programs of the solver's interface (not SOS-derived), for edge-case parity:
    * "free":   no PSD block at all, K = R^t (t = 4, m = 3): min c^T x s.t. A x = b with c = A^T y0, so every
                feasible x is optimal with value y0^T b (closed form);
    * "detached": a planted POP (n = 3) plus a 4 x 4 PSD block that appears in no constraint (ten empty
                orthogonal columns, c = 0 on them): same optimum gamma0, the extra block's iterate stays 0."""
    rng = np.random.default_rng(seed)
    if kind == "free":
        A = rng.standard_normal((3, 4))
        x0, y0 = rng.standard_normal(4), rng.standard_normal(3)
        b = A @ x0
        c = A.T @ y0
        import scipy.sparse as sp_

        return Problem("free", sp_.csc_matrix(A), b, c, 4, [], dict(kind="free", optimum=float(y0 @ b)))
    if kind == "detached":
        base = planted_pop("detached", 3, 2, seed)
        import scipy.sparse as sp_

        A = sp_.hstack([base.A, sp_.csc_matrix((base.m, 10))]).tocsc()
        c = np.concatenate([base.c, np.zeros(10)])
        meta = dict(base.meta)
        meta["kind"] = "detached"
        prob = Problem("detached", A, base.b.copy(), c, base.n_free, list(base.psd_dims) + [4], meta)
        prob.row_expo = base.row_expo
        prob.block_info = base.block_info
        return prob
    raise KeyError(kind)


def univariate_feasibility(name: str, coeffs: list[float]) -> Problem:
    """Is g0(x) = sum_k coeffs[k] x^k SOS?  (SPEC.md S:169-170 examples.)  t = 0."""
    deg = len(coeffs) - 1
    assert deg % 2 == 0
    ex = np.arange(len(coeffs), dtype=np.int64)[:, None]
    g0 = Poly(np.array(coeffs, dtype=float), ex)
    con = SosConstraint(g0=g0, g=[], blocks=[GramBlock(basis(1, 0, deg // 2))])
    return assemble(name, 1, [con], np.zeros(0), dict(kind="univariate"))


def make_config(idx_or_name, seed: int | None = None) -> Problem:
    name = CONFIG_NAMES[idx_or_name] if isinstance(idx_or_name, int) else idx_or_name
    s = DEFAULT_SEEDS[name] if seed is None else seed
    if name == "pop6":
        return planted_pop(name, 6, 3, s)
    if name == "pop20":
        return planted_pop(name, 20, 8, s)
    if name == "pop40":
        return planted_pop(name, 40, 16, s)
    if name == "box24":
        return planted_pop(name, 24, 10, s, box=True)
    if name == "lyap10":
        return lyapunov(name, 10, s)
    raise KeyError(name)


def svec(M: np.ndarray) -> np.ndarray:
    """'U' packed svec with sqrt(2) off-diagonal scaling (layout helper for planted points)."""
    N = M.shape[0]
    ii, jj = svec_pairs(N)
    return np.where(ii == jj, 1.0, SQRT2) * M[ii, jj]


def planted_kkt(prob: Problem):
    """Exact primal-dual optimum of a planted (box) POP as HSDE vectors (SURVEY §8(c) pins).

    X0* = sum_k c_k c_k^T, X_i* = 0; y* = -(x0^alpha)_alpha; Z0* = v2(x0) v2(x0)^T,
    Z_i* = (1 - x0_i^2) v1(x0) v1(x0)^T; gamma* = gamma0, tau = 1, kappa = 0.
    Returns (xi, y, z) with xi = (gamma, svec blocks...), z the dual slack.
    """
    meta = prob.meta
    n = meta["nvars"]
    x0 = np.array(meta["x0"])
    C = np.array(meta["C"])
    row_expo = prob.row_expo
    y = -np.prod(np.power(x0[None, :], row_expo), axis=1)
    xi_parts = [np.array([meta["gamma0"]])]
    z_parts = [np.zeros(1)]
    B2 = basis(n, 0, 2)
    if meta["kind"] == "box_pop":
        B1 = basis(n, 0, 1)
        v1 = np.prod(np.power(x0[None, :], B1), axis=1)
        for i in range(n):
            xi_parts.append(np.zeros(B1.shape[0] * (B1.shape[0] + 1) // 2))
            z_parts.append(svec((1.0 - x0[i] ** 2) * np.outer(v1, v1)))
    v2 = np.prod(np.power(x0[None, :], B2), axis=1)
    xi_parts.append(svec(C.T @ C))
    z_parts.append(svec(np.outer(v2, v2)))
    return np.concatenate(xi_parts), y, np.concatenate(z_parts)


def expected_dims(name: str) -> dict:
    """Closed-form sizes of each config."""
    if name.startswith("pop"):
        n = int(name[3:])
        N = comb(n + 2, 2)
        return dict(m=comb(n + 4, 4), t=1, psd=[N])
    if name == "box24":
        n = 24
        return dict(m=comb(n + 4, 4), t=1, psd=[n + 1] * n + [comb(n + 2, 2)])
    if name == "lyap10":
        return dict(m=1000 + 8007, t=1000, psd=[65, 285])
    raise KeyError(name)
