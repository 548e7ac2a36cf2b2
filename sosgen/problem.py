"""Problem container and SOS -> conic assembly by coefficient matching.

Input-generation code (SURVEY §2 status GEN).  It writes the conic data of PAPER.md
`eq:generalSDP`: A = [A_free | A_psd], b, c, cone dims.  It holds none of the
ADMM arithmetic and is imported by both the oracle tests and the GPU tests as the single
source of problem bytes.

Conventions (readings C1-C4):
* column order: t free columns first, then one svec block per PSD cone;
* svec = LAPACK 'U' packed, column-major: position p(i, j) = i + j(j+1)/2 for i <= j, and
  off-diagonal entries carry the factor sqrt(2) in A (so <B_alpha, X> = a_row . svec(X));
* a row is kept iff it has a nonzero in A or in b (C3);
* coefficient matching: sum over Gram blocks <B_alpha^{(b)}, X_b> + sum_i u_i g_{i,alpha}
  = g_{0,alpha}, i.e. column i of A_free holds g_i's coefficients and b holds g_0's.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .monomials import MonomialIndex

SQRT2 = float(np.sqrt(2.0))


@dataclass
class Poly:
    """Sparse polynomial: coef[r] * x^expo[r]."""

    coef: np.ndarray
    expo: np.ndarray  # (terms x nvars) int

    @staticmethod
    def const(nvars: int, value: float) -> "Poly":
        return Poly(np.array([float(value)]), np.zeros((1, nvars), dtype=np.int64))

    @staticmethod
    def zero(nvars: int) -> "Poly":
        return Poly(np.zeros(0), np.zeros((0, nvars), dtype=np.int64))


@dataclass
class GramBlock:
    """One Gram matrix X_b >= 0 entering a constraint as mult(x) * v_b(x)^T X_b v_b(x)."""

    basis: np.ndarray  # (N x nvars) exponents of v_b in graded-lex order
    mult: Poly | None = None  # weight polynomial p_i of PAPER.md §VI (None = 1)


@dataclass
class SosConstraint:
    """s(x) = g0(x) - sum_i u_i g_i(x), with s = sum_b mult_b v_b^T X_b v_b."""

    g0: Poly
    g: list[Poly]
    blocks: list[GramBlock]


@dataclass
class Problem:
    name: str
    A: sp.csc_matrix
    b: np.ndarray
    c: np.ndarray
    n_free: int
    psd_dims: list[int]
    meta: dict = field(default_factory=dict)
    # generator-side description (not part of the conic data handed to the solvers):
    # row_expo[alpha] = monomial of row alpha; block_info[b] = Gram basis of PSD block b etc.
    row_expo: np.ndarray | None = None
    block_info: list[dict] | None = None

    @property
    def m(self) -> int:
        return self.A.shape[0]

    @property
    def n(self) -> int:
        return self.A.shape[1]

    def save(self, path: str) -> None:
        A = self.A.tocsc()
        A.sort_indices()
        np.savez(path, name=self.name, colptr=A.indptr.astype(np.int64), rowidx=A.indices.astype(np.int32),
                 val=A.data.astype(np.float64), shape=np.array(A.shape, dtype=np.int64), b=self.b, c=self.c,
                 n_free=self.n_free, psd_dims=np.array(self.psd_dims, dtype=np.int32),
                 meta=json.dumps(self.meta))

    @staticmethod
    def load(path: str) -> "Problem":
        z = np.load(path, allow_pickle=False)
        A = sp.csc_matrix((z["val"], z["rowidx"], z["colptr"]), shape=tuple(z["shape"]))
        return Problem(str(z["name"]), A, z["b"], z["c"], int(z["n_free"]), [int(d) for d in z["psd_dims"]],
                       json.loads(str(z["meta"])))


def svec_pairs(N: int) -> tuple[np.ndarray, np.ndarray]:
    """(i, j) of every svec position p in 'U' packed column-major order (i <= j)."""
    jj = np.repeat(np.arange(N, dtype=np.int64), np.arange(1, N + 1))
    ii = np.arange(N * (N + 1) // 2, dtype=np.int64) - jj * (jj + 1) // 2
    return ii, jj


def graded_lex_order(expo: np.ndarray) -> np.ndarray:
    """Permutation sorting exponent rows: degree ascending, then exponents descending lex."""
    expo = np.asarray(expo, dtype=np.int64)
    deg = expo.sum(axis=1)
    keys = [-expo[:, v] for v in range(expo.shape[1] - 1, -1, -1)] + [deg]
    return np.lexsort(keys)


def _unique_rows(expo: np.ndarray) -> np.ndarray:
    e8 = np.ascontiguousarray(np.asarray(expo).astype(np.int8))
    v = e8.view(np.dtype((np.void, e8.shape[1]))).ravel()
    _, idx = np.unique(v, return_index=True)
    return expo[np.sort(idx)]


def _block_terms(blk: GramBlock, nvars: int):
    """(position, exponent, value) triplets of one Gram block's svec columns."""
    N = blk.basis.shape[0]
    ii, jj = svec_pairs(N)
    w = np.where(ii == jj, 1.0, SQRT2)
    mult = blk.mult if blk.mult is not None else Poly.const(nvars, 1.0)
    pos, ex, val = [], [], []
    base = blk.basis[ii] + blk.basis[jj]
    for coef, e in zip(mult.coef, mult.expo):
        pos.append(np.arange(len(ii)))
        ex.append(base + e[None, :])
        val.append(w * coef)
    return np.concatenate(pos), np.concatenate(ex), np.concatenate(val)


def assemble(name: str, nvars: int, constraints: list[SosConstraint], w: np.ndarray, meta: dict | None = None) -> Problem:
    """Coefficient matching for k SOS constraints sharing u."""
    t = len(w)
    for con in constraints:
        if len(con.g) != t:
            raise ValueError("every constraint needs t polynomials g_i")
    rows_all, cols_all, vals_all = [], [], []
    b_all = []
    row_off = 0
    psd_dims: list[int] = []
    block_info: list[dict] = []
    col_off = t
    row_expo_all = []
    # first pass: per-constraint row sets
    for con in constraints:
        terms = [_block_terms(blk, nvars) for blk in con.blocks]
        cand = [con.g0.expo[con.g0.coef != 0]] + [g.expo[g.coef != 0] for g in con.g] + [tr[1] for tr in terms]
        cand = [c_.reshape(-1, nvars) for c_ in cand if len(c_)]
        allx = _unique_rows(np.concatenate(cand, axis=0)) if cand else np.zeros((0, nvars), dtype=np.int64)
        rows_expo = allx[graded_lex_order(allx)]
        idx = MonomialIndex(rows_expo)
        m_j = rows_expo.shape[0]
        # b
        bj = np.zeros(m_j)
        if len(con.g0.coef):
            np.add.at(bj, idx.lookup(con.g0.expo), con.g0.coef)
        b_all.append(bj)
        # free columns: g_i coefficients
        for i, g in enumerate(con.g):
            if len(g.coef) == 0:
                continue
            r = idx.lookup(g.expo)
            rows_all.append(r + row_off)
            cols_all.append(np.full(len(r), i))
            vals_all.append(g.coef.astype(np.float64))
        # PSD blocks
        for blk, (pos, ex, val) in zip(con.blocks, terms):
            N = blk.basis.shape[0]
            r = idx.lookup(ex)
            assert (r >= 0).all()
            rows_all.append(r + row_off)
            cols_all.append(pos + col_off)
            vals_all.append(val)
            psd_dims.append(N)
            block_info.append(dict(constraint=len(row_expo_all), row_offset=row_off,
                                   weighted=blk.mult is not None, basis=blk.basis))
            col_off += N * (N + 1) // 2
        row_expo_all.append(rows_expo)
        row_off += m_j
    m, n = row_off, col_off
    A = sp.coo_matrix((np.concatenate(vals_all), (np.concatenate(rows_all), np.concatenate(cols_all))),
                      shape=(m, n)).tocsc()
    A.sum_duplicates()
    A.eliminate_zeros()
    b = np.concatenate(b_all)
    c = np.zeros(n)
    c[:t] = w
    meta = dict(meta or {})
    meta.setdefault("nvars", nvars)
    prob = Problem(name, A, b, c, t, psd_dims, meta)
    prob.row_expo = np.concatenate(row_expo_all, axis=0)
    prob.block_info = block_info
    return prob
