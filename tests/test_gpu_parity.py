"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Criteria (BASELINE.json north_star; readings C9, C13):
* alpha-map and D bit-exact against brute-force enumeration (Proposition 1);
* affine projection and PSD projection against the oracle's routines on identical inputs;
* per-iterate relative error <= 1e-9 over the first 20 iterations, normalised by ||(u, v)|| of the
  oracle iterate (reading C13);
* residual-stop iteration counts within +-2% and the converged objective within 1e-6 relative.
"""
import numpy as np
import pytest

from oracle import HsdeOracle, Status, brute_force_structure, proj_psd_svec, svec
from sosgen import ball_pop, make_config, planted_kkt, unbounded_pop, univariate_feasibility
from sosgen.configs import planted_pop
from sosgen.matrix_sos import brute_force_counts, matrix_planted_kkt, matrix_sos_pop

pytestmark = pytest.mark.gpu

SMALL = ["pop6", "sq", "neg", "one", "pop3k2", "ball4", "msos2", "pop8", "unb6", "free", "detached"]
LARGE = ["pop20", "lyap10", "box24", "pop40", "msos3", "unb10"]


def make(name):
    if name == "sq":
        return univariate_feasibility("sq", [1.0, 2.0, 1.0])
    if name == "neg":
        return univariate_feasibility("neg", [-1.0, 0.0, -1.0])
    if name == "one":  # degenerate: a 1 x 1 PSD block, t = 0, m = 1
        return univariate_feasibility("one", [1.0])
    if name == "pop3k2":
        return planted_pop("pop3k2", 3, 2, seed=5)
    if name == "ball4":
        return ball_pop(4)
    if name == "pop8":  # N = 45: the CTA-per-block Jacobi (33 <= N <= 64); N <= 32 use one warp per block
        return planted_pop("pop8", 8, 4, seed=2)
    if name == "msos2":  # matrix-valued SOS (Proposition 2): Y in S^{2 * 10} (Jacobi path)
        return matrix_sos_pop("msos2", 3, 2, 2, 2, seed=3)
    if name == "msos3":  # Y in S^{3 * 28} (cluster tridiagonalisation path)
        return matrix_sos_pop("msos3", 6, 3, 2, 3, seed=4)
    if name in ("free", "detached"):  # degenerate: no PSD block / a block in no constraint (empty columns)
        from sosgen.configs import edge_program

        return edge_program(name)
    if name.startswith("unb"):  # dual infeasible (unbounded) program: N = 28 (Jacobi) / 66 (large-block path)
        return unbounded_pop(name, int(name[3:]))
    return make_config(name)


@pytest.fixture(scope="module")
def solvers():
    from paper_1708_04174_b200 import SosAdmm

    cache = {}

    def get(name, **kw):
        key = (name, tuple(sorted(kw.items())))
        if key not in cache:
            prob = make(name)
            cache[key] = (prob, SosAdmm.from_problem(prob, **kw), HsdeOracle.from_problem(prob))
        return cache[key]

    yield get
    for _, s, _ in cache.values():
        s.close()


@pytest.mark.parametrize("name", SMALL + LARGE)
def test_structure_bit_exact(name, solvers):
    prob, gpu, _ = solvers(name)
    row_of, D, tl = gpu.get_structure()
    if name.startswith("msos"):  # Proposition 2: D = ordered-pair counts of every (alpha, i, j) row
        assert np.array_equal(D, brute_force_counts(prob).astype(np.float64))
        assert np.all(row_of[prob.n_free:] >= 0) and tl == prob.n_free
        return
    if name in ("free", "detached"):  # generator-made, not SOS-assembled: structure from A directly
        A = prob.A.tocsc()
        cnt = np.diff(A.indptr)
        exp_row = np.full(prob.n, -2)
        for j in range(prob.n_free, prob.n):
            exp_row[j] = A.indices[A.indptr[j]] if cnt[j] == 1 else (-1 if cnt[j] == 0 else -2)
        assert np.array_equal(row_of.astype(np.int64)[prob.n_free:], exp_row[prob.n_free:])
        Dref = np.zeros(prob.m)
        for j in range(prob.n_free, prob.n):
            if cnt[j] == 1:
                v = A.data[A.indptr[j]]
                Dref[A.indices[A.indptr[j]]] += 1.0 if abs(v) == 1.0 else (2.0 if abs(v) == np.sqrt(2.0) else v * v)
        assert np.array_equal(D, Dref)
        return
    maps, n_alpha = brute_force_structure(prob.row_expo, prob.block_info, prob.m)
    assert np.array_equal(D, n_alpha.astype(np.float64))  # exact integers
    off = prob.n_free
    n_weighted = 0
    for N, amap, info in zip(prob.psd_dims, maps, prob.block_info):
        L = N * (N + 1) // 2
        if amap is None:
            assert np.all(row_of[off:off + L] == -2)
            n_weighted += L
        else:
            assert np.array_equal(row_of[off:off + L].astype(np.int64), amap)
        off += L
    assert tl == prob.n_free + n_weighted


@pytest.mark.parametrize("name", SMALL + LARGE)
def test_affine_projection_parity(name, solvers):
    prob, gpu, orc = solvers(name)
    rng = np.random.default_rng(11)
    for _ in range(3):
        w1, w2, w3 = rng.standard_normal(prob.n), rng.standard_normal(prob.m), float(rng.standard_normal())
        g1, g2, g3 = gpu.project_affine(w1, w2, w3)
        o1, o2, o3 = orc.affine(w1, w2, w3)
        ref = np.concatenate([o1, o2, [o3]])
        got = np.concatenate([g1, g2, [g3]])
        # both sides round the same cancellations: relative 1e-10 of |w| + |u|
        assert np.linalg.norm(got - ref) <= 1e-10 * (np.linalg.norm(ref) + np.linalg.norm(w1) + np.linalg.norm(w2))


@pytest.mark.parametrize("name", SMALL + LARGE)
def test_psd_projection_parity(name, solvers):
    prob, gpu, _ = solvers(name)
    rng = np.random.default_rng(3)
    nb = len(prob.psd_dims)
    for bidx in sorted({0, 1, 2, nb - 1} & set(range(nb))):
        N = prob.psd_dims[bidx]
        L = N * (N + 1) // 2
        for kind in ["gauss", "lowrank", "zero", "psd", "nsd"]:
            if kind == "gauss":
                a = rng.standard_normal(L)
            elif kind == "zero":  # degenerate: Pi(0) = 0
                a = np.zeros(L)
            elif kind in ("psd", "nsd"):  # already in the cone: Pi = identity / Pi = 0
                G = rng.standard_normal((N, N))
                a = svec((1.0 if kind == "psd" else -1.0) * (G @ G.T + np.eye(N)))
            else:  # clustered spectrum: rank-3 PSD minus rank-2 PSD plus tiny noise
                G = rng.standard_normal((N, 3))
                H = rng.standard_normal((N, 2))
                X = G @ G.T - H @ H.T + 1e-10 * np.eye(N)
                a = svec(X)
            got = gpu.project_psd(bidx, a)
            ref = proj_psd_svec(a, N)
            assert np.linalg.norm(got - ref) <= 1e-11 * max(np.linalg.norm(a), 1e-300), (bidx, N, kind)


def _rel(a, b, scale):
    return np.linalg.norm(a - b) / scale


@pytest.mark.parametrize("name", SMALL + LARGE)
def test_first_20_iterates(name, solvers):
    prob, gpu, orc = solvers(name)
    gpu.set_iterate(np.zeros(prob.n), np.zeros(prob.m), np.zeros(prob.n), None, 1.0, 0.0, 0)
    st = orc.initial_state()
    worst_u = worst_v = 0.0
    worst_part = (0.0, "")
    for k in range(1, 21):
        st = orc.step(st)
        gpu.iterate(1)
        g = gpu.get_iterate()
        if g["iter"] != k:  # terminated early (tiny problems); test_convergence_parity covers status
            break
        ug = np.concatenate([g["xi"], g["y"], [g["tau"]]])
        vg = np.concatenate([g["z"], g["s"], [g["kappa"]]])
        scale = np.linalg.norm(np.concatenate([st.u(), st.v()]))
        worst_u = max(worst_u, _rel(ug, st.u(), scale))
        worst_v = max(worst_v, _rel(vg, st.v(), scale))
        # per component (tau ~ 2e-6 at k = 1 on pop20 is invisible in the joint norm): tau, kappa,
        # the free part, y and every PSD block of xi and z, each relative to its own size, with an absolute
        # floor of 1e-12 of the joint norm for parts that are (near) zero on both sides
        parts = [("tau", [g["tau"]], [st.tau]), ("kappa", [g["kappa"]], [st.kappa]), ("y", g["y"], st.y),
                 ("xi_free", g["xi"][:prob.n_free], st.xi[:prob.n_free])]
        off = prob.n_free
        for bi, N in enumerate(prob.psd_dims):
            L = N * (N + 1) // 2
            parts.append((f"xi_{bi}", g["xi"][off:off + L], st.xi[off:off + L]))
            parts.append((f"z_{bi}", g["z"][off:off + L], st.z[off:off + L]))
            off += L
        for pname, a, b in parts:
            a, b = np.asarray(a), np.asarray(b)
            err = np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-3 * scale)
            if err > worst_part[0]:
                worst_part = (err, f"{pname}@k={k}")
            assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b) + 1e-12 * scale, (pname, k, a[:3], b[:3])
    assert worst_u <= 1e-9 and worst_v <= 1e-9, (worst_u, worst_v)


@pytest.mark.parametrize("name", ["pop6", "sq", "neg", "pop3k2", "ball4", "msos2", "unb6", "unb10", "free", "detached"])
def test_convergence_parity(name, solvers):
    prob, gpu, orc = solvers(name, tol=1e-4, max_iters=5000)
    st, status, hist = orc.solve(tol=1e-4, max_iters=5000)
    gpu.set_iterate(np.zeros(prob.n), np.zeros(prob.m), np.zeros(prob.n), None, 1.0, 0.0, 0)
    info = gpu.iterate(5000)
    assert info["status"] == int(status)
    assert abs(info["iter"] - st.k) <= max(1, int(0.02 * st.k))
    if status == Status.OPTIMAL and np.isfinite(hist[-1][3]) and hist[-1][3] != 0:
        assert abs(info["pobj"] - hist[-1][3]) <= 1e-6 * abs(hist[-1][3])


@pytest.mark.parametrize("name", ["pop6", "pop20", "box24", "pop40", "msos2", "msos3"])
def test_planted_fixed_point(name, solvers):
    prob, gpu, _ = solvers(name)
    xi, y, z = matrix_planted_kkt(prob) if name.startswith("msos") else planted_kkt(prob)
    gpu.set_iterate(xi, y, z, None, 1.0, 0.0, 0)
    gpu.iterate(1)
    g = gpu.get_iterate()
    scale = np.linalg.norm(np.concatenate([xi, y, [1.0], z]))
    assert np.linalg.norm(g["xi"] - xi) <= 1e-12 * scale
    assert np.linalg.norm(g["z"] - z) <= 1e-12 * scale
    assert np.linalg.norm(g["y"] - y) <= 1e-12 * scale
    assert abs(g["tau"] - 1.0) <= 1e-12 and abs(g["kappa"]) <= 1e-12


@pytest.mark.parametrize("name", ["unb6", "unb10"])
def test_dual_infeasible_certificate(name, solvers):
    """DUAL_INFEASIBLE: the GPU's final xi is a certificate — xi in K,
    c^T xi < 0, |A xi| <= tol (-c^T xi) — and tau = 0 < kappa, as on the oracle."""
    prob, gpu, _ = solvers(name, tol=1e-4, max_iters=5000)
    gpu.set_iterate(np.zeros(prob.n), np.zeros(prob.m), np.zeros(prob.n), None, 1.0, 0.0, 0)
    info = gpu.iterate(5000)
    assert info["status_name"] == "DUAL_INFEASIBLE", info
    g = gpu.get_iterate()
    cx = prob.c @ g["xi"]
    assert cx < 0 and np.linalg.norm(prob.A @ g["xi"]) <= 1e-4 * (-cx)
    assert g["tau"] == 0.0 and g["kappa"] > 0.0
    N = prob.psd_dims[0]
    X = np.zeros((N, N))
    q = 0
    for j in range(N):
        for i in range(j + 1):
            X[i, j] = X[j, i] = g["xi"][1 + q] / (1.0 if i == j else np.sqrt(2.0))
            q += 1
    assert np.linalg.eigvalsh(X).min() >= -1e-10 * np.abs(X).max()


def test_nonfinite_iterate_reported():
    """a non-finite iterate stops the solve with E_NONFINITE naming the iteration; the
    error is latched (every later call returns it)."""
    from paper_1708_04174_b200 import SosAdmm

    prob = make_config("pop6")
    gpu = SosAdmm.from_problem(prob, tol=1e-4, max_iters=100)
    try:
        xi = np.zeros(prob.n)
        xi[5] = np.nan
        gpu.set_iterate(xi, np.zeros(prob.m), np.zeros(prob.n), None, 1.0, 0.0, 0)
        with pytest.raises(RuntimeError, match="non-finite"):
            gpu.iterate(10)
        with pytest.raises(RuntimeError, match="non-finite"):
            gpu.iterate(1)
    finally:
        gpu.close()


def test_first_iterates_near_max_block():
    """Near the largest supported block (SOSADMM_MAX_BLOCK = 1280): a planted POP with n = 48 (Gram
    N = C(50, 2) = 1225, m = C(52, 4) = 270,725; every cluster CTA at its largest row share), 5 iterates
    against the oracle at the reading-C13 bar, plus the per-block check of xi and z."""
    from paper_1708_04174_b200 import SosAdmm

    prob = planted_pop("pop48", 48, 19, seed=2)
    assert prob.psd_dims == [1225] and prob.m == 270725
    gpu = SosAdmm.from_problem(prob, tol=1e-300, max_iters=1 << 40)
    orc = HsdeOracle.from_problem(prob)
    st = orc.initial_state()
    try:
        for k in range(1, 6):
            st = orc.step(st)
            gpu.iterate(1)
            g = gpu.get_iterate()
            ug = np.concatenate([g["xi"], g["y"], [g["tau"]]])
            vg = np.concatenate([g["z"], g["s"], [g["kappa"]]])
            scale = np.linalg.norm(np.concatenate([st.u(), st.v()]))
            assert _rel(ug, st.u(), scale) <= 1e-9 and _rel(vg, st.v(), scale) <= 1e-9, k
            blk = slice(prob.n_free, prob.n)
            assert np.linalg.norm(g["xi"][blk] - st.xi[blk]) <= 1e-8 * np.linalg.norm(st.xi[blk]) + 1e-12 * scale
            assert np.linalg.norm(g["z"][blk] - st.z[blk]) <= 1e-8 * np.linalg.norm(st.z[blk]) + 1e-12 * scale
    finally:
        gpu.close()
