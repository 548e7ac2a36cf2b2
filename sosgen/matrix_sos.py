"""Matrix-valued SOS programs (§V, `E:matrixSOS` P:503-506, `E:matrixSOSprogram`
P:508-515, Proposition 2) — input generation only.

P(x) = P_0(x) - sum_h u_h P_h(x) (r x r symmetric polynomial matrices) is an SOS matrix iff
P(x) = (I_r (x) v_d(x))^T Y (I_r (x) v_d(x)) with Y in S^{rN}_+ (P:503-506).  Coefficient matching
gives one equation per triple (alpha, i, j): <Y_ij, B_alpha> = (C_alpha(u))_ij.

Conventions of this assembly (reading C16):
* Y is one PSD block of size l = r N, index a = i N + beta (block-row i, basis monomial beta);
  its svec columns follow the scalar convention ('U' packed, sqrt(2) off the diagonal);
* only triples with i <= j are kept (C_alpha and Y are symmetric, the (alpha, j, i) equation
  repeats the (alpha, i, j) one); rows ordered by (i, j) lexicographically, then alpha graded-lex;
* an off-diagonal-block equation (i < j) is multiplied by sqrt(2), so every svec column of Y
  carries the coefficient 1 (i < j) or the scalar-case 1 / sqrt(2) pattern (i = j) and
  A2 A2^T = diag(n_alpha) with the same integer counts as Proposition 1 (Proposition 2: the rows
  of A2 are orthogonal; this scaling only fixes the diagonal).

Planted instance (closed-form optimum, like the scalar planted POP): H(x) in R^{K x r} with entries
of degree <= d, H(x0) = 0, P(x) = gamma0 I_r + H(x)^T H(x);  max gamma s.t. P(x) - gamma I_r SOS
has optimum gamma0 (P - gamma0 I = H^T H is an SOS matrix; P(x0) - gamma I >= 0 forces gamma <=
gamma0).  Seeded draw order: x0 ~ N(0, I_n), then the coefficients of H (K x r x N, N(0, 1)).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .monomials import MonomialIndex, basis_tuples, exponents
from .problem import Problem, graded_lex_order

SQRT2 = float(np.sqrt(2.0))


def matrix_sos_pop(name: str, nvars: int, r: int, d: int, K: int, seed: int, gamma0: float = 1.0) -> Problem:
    rng = np.random.default_rng(seed)
    x0 = rng.standard_normal(nvars)
    B = exponents(basis_tuples(nvars, 0, d), nvars)  # v_d, graded-lex
    N = B.shape[0]
    Hc = rng.standard_normal((K, r, N))
    vx0 = np.prod(np.power(x0[None, :], B), axis=1)
    Hc[:, :, 0] -= Hc @ vx0  # H(x0) = 0 (basis entry 0 is the constant monomial)
    # rows: monomials of degree <= 2d
    R = exponents(basis_tuples(nvars, 0, 2 * d), nvars)
    R = R[graded_lex_order(R)]
    ridx = MonomialIndex(R)
    mA = R.shape[0]
    pairs = [(i, j) for i in range(r) for j in range(i, r)]
    row_of_pair = {p: k * mA for k, p in enumerate(pairs)}
    m = mA * len(pairs)
    # P_0 coefficients: gamma0 I + sum_k H_k^T H_k, H_k(x) = Hc[k] v(x)  ->  (i, j) entry
    # sum_k sum_{beta, gamma} Hc[k, i, beta] Hc[k, j, gamma] x^(beta + gamma)
    b = np.zeros(m)
    bb, gg = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    ex = B[bb.ravel()] + B[gg.ravel()]
    rows_ex = ridx.lookup(ex)
    for (i, j) in pairs:
        off = row_of_pair[(i, j)]
        coef = np.einsum("kb,kc->bc", Hc[:, i, :], Hc[:, j, :]).ravel()
        np.add.at(b, off + rows_ex, coef)
        if i == j:
            b[off + ridx.lookup(np.zeros((1, nvars), dtype=np.int64))[0]] += gamma0
    # free column: P_1 = I_r (u = gamma enters as P_0 - gamma I)
    rows, cols, vals = [], [], []
    const_row = ridx.lookup(np.zeros((1, nvars), dtype=np.int64))[0]
    for i in range(r):
        rows.append(row_of_pair[(i, i)] + const_row)
        cols.append(0)
        vals.append(1.0)
    # Y columns: svec over a = i N + beta, position p(a1, a2) = a1 + a2 (a2 + 1) / 2 for a1 <= a2
    L = r * N
    col = 1
    for a2 in range(L):
        i2, g2 = divmod(a2, N)
        for a1 in range(a2 + 1):
            i1, g1 = divmod(a1, N)
            alpha_row = ridx.lookup((B[g1] + B[g2])[None, :])[0]
            if i1 == i2:
                v = 1.0 if g1 == g2 else SQRT2
            else:
                v = 1.0  # the (alpha, i1, i2) equation scaled by sqrt(2): sqrt(2) * (1 / sqrt(2))
            rows.append(row_of_pair[(min(i1, i2), max(i1, i2))] + alpha_row)
            cols.append(col)
            vals.append(v)
            col += 1
    # scale the off-diagonal-block right-hand sides by sqrt(2) like their rows
    for (i, j) in pairs:
        if i < j:
            b[row_of_pair[(i, j)]:row_of_pair[(i, j)] + mA] *= SQRT2
    A = sp.coo_matrix((np.array(vals), (np.array(rows), np.array(cols))), shape=(m, 1 + L * (L + 1) // 2)).tocsc()
    A.sum_duplicates()
    # keep rows with a nonzero in A or b (reading C3)
    keep = np.flatnonzero((np.abs(A).sum(axis=1).A.ravel() != 0) | (b != 0))
    A = A[keep].tocsc()
    b = b[keep]
    c = np.zeros(A.shape[1])
    c[0] = -1.0  # min -gamma
    meta = dict(kind="matrix_sos_pop", nvars=nvars, r=r, d=d, K=K, seed=seed, gamma0=gamma0, x0=x0.tolist())
    prob = Problem(name, A, b, c, 1, [L], meta)
    prob.row_expo = None
    prob.block_info = [dict(kind="matrix", r=r, basis=B, rows=R, pairs=pairs, keep=keep)]
    return prob


def brute_force_counts(prob: Problem) -> np.ndarray:
    """Expected diagonal of A2 A2^T from the definition: for row (alpha, i, j), the number of ORDERED
    basis pairs (beta, gamma) with beta + gamma = alpha (Proposition 2's n_alpha), by enumeration."""
    info = prob.block_info[0]
    B, R, pairs, keep = info["basis"], info["rows"], info["pairs"], info["keep"]
    cnt = {}
    for x in B:
        for y in B:
            key = tuple(int(v) for v in x + y)
            cnt[key] = cnt.get(key, 0) + 1
    full = np.zeros(len(pairs) * R.shape[0], dtype=np.int64)
    for k, _ in enumerate(pairs):
        for a in range(R.shape[0]):
            full[k * R.shape[0] + a] = cnt.get(tuple(int(v) for v in R[a]), 0)
    return full[keep]


def matrix_planted_kkt(prob: Problem):
    """Exact primal-dual optimum of the planted matrix SOS program (closed form, no solver):
    Y* = sum_k h_k h_k^T (h_k[(i, beta)] = H[k, i, beta], so (I (x) v)^T Y* (I (x) v) = H^T H),
    gamma = gamma0;  dual: Z* = (I_r (x) v(x0)) (I_r / r) (I_r (x) v(x0))^T (point evaluation at x0,
    <Y*, Z*> = sum_k |H_k(x0)|^2 / r = 0), y*_(alpha,i,i) = -x0^alpha / r, y*_(alpha,i,j<i) = 0,
    z* = [0; svec(Z*)] (A_free^T y* = -sum_i x0^0 / r * 1 = -1 = c_gamma)."""
    from .configs import svec  # layout helper

    meta, info = prob.meta, prob.block_info[0]
    rng = np.random.default_rng(meta["seed"])
    nvars, r, K = meta["nvars"], meta["r"], meta["K"]
    B, R, pairs, keep = info["basis"], info["rows"], info["pairs"], info["keep"]
    N = B.shape[0]
    x0 = rng.standard_normal(nvars)
    Hc = rng.standard_normal((K, r, N))
    vx0 = np.prod(np.power(x0[None, :], B), axis=1)
    Hc[:, :, 0] -= Hc @ vx0
    cols = Hc.reshape(K, r * N)  # index i N + beta
    Y = cols.T @ cols
    xi = np.concatenate([[meta["gamma0"]], svec(Y)])
    vI = np.kron(np.eye(r), vx0[:, None])  # (rN x r)
    Z = vI @ vI.T / r
    z = np.concatenate([[0.0], svec(Z)])
    mA = R.shape[0]
    xR = np.prod(np.power(x0[None, :], R), axis=1)
    y = np.zeros(len(pairs) * mA)
    for k, (i, j) in enumerate(pairs):
        if i == j:
            y[k * mA:(k + 1) * mA] = -xR / r
    return xi, y[keep], z
