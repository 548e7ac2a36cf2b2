"""Spectrum of the PSD-projection input over an ADMM run (config 4): counts of positive / negative
eigenvalues and the smaller side r (via the oracle's eigh on the GPU iterate: a = xi - z is the
projection input of the NEXT iteration's block, and xi = Pi(a), z = Pi(a) - a)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1708_04174_b200 import SosAdmm  # noqa: E402
from sosgen import make_config  # noqa: E402

prob = make_config(sys.argv[1] if len(sys.argv) > 1 else "pop40")
g = SosAdmm.from_problem(prob, tol=1e-300, max_iters=1 << 40)
N = prob.psd_dims[0]
ii, jj = np.triu_indices(N)
done = 0
for target in [1, 5, 20, 100, 300, 1000, 3000, 6000, 9000]:
    g.iterate(target - done)
    done = target
    it = g.get_iterate()
    xs = it["xi"][prob.n_free:prob.n_free + N * (N + 1) // 2]
    zs = it["z"][prob.n_free:prob.n_free + N * (N + 1) // 2]
    def unsvec(v):
        M = np.zeros((N, N))
        # 'U' packed column-major: position p(i, j) = i + j (j + 1) / 2
        jidx = np.repeat(np.arange(N), np.arange(1, N + 1))
        iidx = np.arange(len(v)) - jidx * (jidx + 1) // 2
        w = np.where(iidx == jidx, 1.0, 1.0 / np.sqrt(2))
        M[iidx, jidx] = v * w
        M[jidx, iidx] = v * w
        return M
    a = unsvec(xs) - unsvec(zs)  # a = Pi(a) - (Pi(a) - a)
    lam = np.linalg.eigvalsh(a)
    nrm = np.abs(lam).max()
    pos, neg = (lam > 1e-14 * nrm).sum(), (lam < -1e-14 * nrm).sum()
    small = (np.abs(lam) < 1e-8 * nrm).sum()
    print(f"iter {target:5d}: #pos {pos:4d} #neg {neg:4d} r = {min(pos, neg):4d}  |lam| < 1e-8 max: {small:4d}  "
          f"smallest pos {lam[lam > 0].min() if pos else 0:.2e}  largest neg {lam[lam < 0].max() if neg else 0:.2e}", flush=True)
