"""Oracle pins: partial-orthogonality structure (Proposition 1)."""
import json
import os
from math import comb

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import brute_force_structure
from sosgen import ball_pop, expected_dims, make_config, univariate_feasibility
from sosgen.configs import basis
from sosgen.problem import GramBlock, Poly, SosConstraint, assemble

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _orth_cols(prob):
    """Column ranges of the unweighted PSD blocks."""
    off = prob.n_free
    out = []
    for N, info in zip(prob.psd_dims, prob.block_info):
        L = N * (N + 1) // 2
        if not info["weighted"]:
            out.append((off, off + L, N))
        off += L
    return out


def test_n1_d1_counts_match_spec_example():
    g = json.load(open(os.path.join(GOLD, "prop1_n1d1.json")))
    prob = univariate_feasibility("sq", [1.0, 2.0, 1.0])
    maps, n_alpha = brute_force_structure(prob.row_expo, prob.block_info, prob.m)
    assert n_alpha.tolist() == g["D"]
    assert (1 + n_alpha).tolist() == g["P"]


@pytest.mark.parametrize("name", ["pop6", "pop20", "box24", "lyap10"])
def test_bruteforce_matches_assembled_A(name):
    prob = make_config(name)
    maps, n_alpha = brute_force_structure(prob.row_expo, prob.block_info, prob.m)
    A = prob.A.tocsc()
    for (lo, hi, N), amap in zip(_orth_cols(prob), [m_ for m_ in maps if m_ is not None]):
        sub = A[:, lo:hi]
        nnz = np.diff(sub.indptr)
        assert (nnz == 1).all()  # indicator columns are 1-sparse
        assert np.array_equal(sub.indices, amap)  # the assembled row of every svec column
        # sum_alpha n_alpha = N^2 per block (every ordered pair lands in exactly one B_alpha)
        cnt = np.bincount(amap, minlength=prob.m)
        assert cnt.sum() == N * (N + 1) // 2
    total = sum(N * N for (_, _, N) in _orth_cols(prob))
    assert n_alpha.sum() == total


@pytest.mark.parametrize("name", ["pop6", "pop20", "box24", "lyap10"])
def test_prop1_A2A2T_diagonal_equals_counts(name):
    """A_orth A_orth^T is exactly diagonal (off-diagonal entries are structurally 0) and its
    diagonal equals n_alpha up to the rounding of fl(sqrt 2)^2 (reading C10)."""
    prob = make_config(name)
    _, n_alpha = brute_force_structure(prob.row_expo, prob.block_info, prob.m)
    cols = np.concatenate([np.arange(lo, hi) for (lo, hi, _) in _orth_cols(prob)])
    A2 = prob.A.tocsc()[:, cols]
    G = (A2 @ A2.T).tocoo()
    off = G.row != G.col
    assert np.all(G.data[off] == 0.0)
    d = np.zeros(prob.m)
    d[G.row[~off]] = G.data[~off]
    assert np.max(np.abs(d - n_alpha)) <= 4 * np.finfo(float).eps * max(1, n_alpha.max())


@pytest.mark.parametrize("seed", range(6))
def test_prop1_random_scalar_sos(seed):
    """SPEC acceptance 1: random scalar SOS assemblies are partially orthogonal."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 5))
    d = int(rng.integers(1, 3))
    t = int(rng.integers(0, 4))
    B = basis(n, 0, d)
    ex = basis(n, 0, 2 * d)
    g0 = Poly(rng.standard_normal(ex.shape[0]), ex)
    g = [Poly(rng.standard_normal(ex.shape[0]), ex) for _ in range(t)]
    prob = assemble("rnd", n, [SosConstraint(g0, g, [GramBlock(B)])], rng.standard_normal(t))
    assert prob.m == comb(n + 2 * d, 2 * d)
    _, n_alpha = brute_force_structure(prob.row_expo, prob.block_info, prob.m)
    A2 = prob.A.tocsc()[:, t:]
    G = (A2 @ A2.T).toarray()
    assert np.all(G[~np.eye(prob.m, dtype=bool)] == 0.0)
    assert np.max(np.abs(np.diag(G) - n_alpha)) < 1e-14 * max(1, n_alpha.max())


def test_pop40_counts():
    """Config 4 (the headline): 135,751 rows, n_alpha in [1, 6]."""
    prob = make_config("pop40")
    assert prob.m == comb(44, 4) and prob.psd_dims == [861]
    _, n_alpha = brute_force_structure(prob.row_expo, prob.block_info, prob.m)
    assert n_alpha.sum() == 861 ** 2
    assert n_alpha.min() == 1 and n_alpha.max() == 6


@pytest.mark.parametrize("name", ["pop6", "pop20", "box24", "lyap10", "pop40"])
def test_config_dims(name):
    prob = make_config(name)
    ed = expected_dims(name)
    assert prob.m == ed["m"] and prob.n_free == ed["t"] and prob.psd_dims == ed["psd"]


def test_lyap10_lowrank_nnz():
    """config 2's A_1 has 528,900 nonzeros; A has 571,800."""
    prob = make_config("lyap10")
    A = prob.A.tocsc()
    assert A[:, :prob.n_free].nnz == 528900
    assert A.nnz == 571800


@pytest.mark.parametrize("n", [10, 12, 14, 17])
def test_ball_pop_dims_match_table1(n):
    """Table I: N = C(n+2,2); our m keeps the constant row (reading C4): m = m_paper + 1;
    the multiplier Gram is the paper's factorized block: t' - 1 = t_paper (reading C5)."""
    g = json.load(open(os.path.join(GOLD, "table2_ball_pop.json")))["table1_dims"]["rows"]
    Np, mp, tp = g[str(n)]
    prob = ball_pop(n)
    assert prob.psd_dims[-1] == Np
    assert prob.m == mp + 1
    N1 = prob.psd_dims[0]
    assert N1 * (N1 + 1) // 2 == tp
