"""Matrix-valued SOS programs (§V, Proposition 2): the
generator's A2 has orthogonal rows with the integer counts of Proposition 2 (brute force), the
planted closed-form KKT point is an exact fixed point of the oracle's HSDE-ADMM, and the oracle
converges to the planted optimum gamma0.  The CUDA path on the same programs: tests/test_gpu_parity.py."""
from math import comb

import numpy as np

from oracle import HsdeOracle, OracleState, Status
from sosgen.matrix_sos import brute_force_counts, matrix_planted_kkt, matrix_sos_pop


def test_proposition2_structure():
    for (n, r, d, K) in [(3, 2, 1, 2), (4, 3, 2, 2), (2, 4, 1, 3)]:
        p = matrix_sos_pop("msos", n, r, d, K, seed=1)
        A2 = p.A.tocsc()[:, 1:]
        # every column of Y has exactly one nonzero: rows pairwise orthogonal (Proposition 2)
        assert np.all(np.diff(A2.indptr) == 1)
        G = (A2 @ A2.T).tocoo()
        assert np.all(G.row == G.col)
        # diagonal = ordered-pair counts n_alpha of the row's (alpha, i, j) (to the rounding of
        # fl(sqrt 2)^2 = 2 + 4.4e-16 on the i = j blocks)
        assert np.allclose(np.asarray(A2.multiply(A2).sum(axis=1)).ravel(), brute_force_counts(p), rtol=0, atol=1e-14)
        assert p.psd_dims == [r * comb(n + d, d)]  # Y in S^{r N}, N = C(n + d, d)


def test_planted_matrix_kkt_is_fixed_point():
    p = matrix_sos_pop("msos", 3, 2, 1, 2, seed=0)
    o = HsdeOracle.from_problem(p)
    xi, y, z = matrix_planted_kkt(p)
    st = OracleState(xi, y, 1.0, z, np.zeros(p.m), 0.0)
    res = o.residuals(st)
    assert res.pres < 1e-13 and res.dres < 1e-13 and res.gap < 1e-12
    st2 = o.step(st)
    nuv = np.linalg.norm(np.concatenate([st.u(), st.v()]))
    assert np.linalg.norm(st2.u() - st.u()) <= 1e-12 * nuv
    assert np.linalg.norm(st2.v() - st.v()) <= 1e-12 * nuv


def test_matrix_sos_optimum_is_gamma0():
    p = matrix_sos_pop("msos", 3, 2, 1, 2, seed=0)
    o = HsdeOracle.from_problem(p)
    st, status, hist = o.solve(tol=1e-8, max_iters=20000)
    assert status == Status.OPTIMAL
    assert abs(-hist[-1][3] - 1.0) < 1e-5
