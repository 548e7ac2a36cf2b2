"""CPU probe (not on any product path): sweeps of the kernel's parallel-order Jacobi on the PSD
projection inputs of real ADMM iterations, cold (V0 = I) vs warm-started (B = V_prev^T A V_prev)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import HsdeOracle  # noqa: E402
from oracle.psd import smat  # noqa: E402
from sosgen import make_config  # noqa: E402

EPS = 2.220446049250313e-16


def pairs(Np, r):
    M = Np - 1
    out = [(M, r % M)]
    for k in range(1, Np // 2):
        out.append(((r + k) % M, (r - k + M) % M))
    return out


def jacobi(A):
    N = A.shape[0]
    Np = N + (N & 1)
    A = np.pad(A, ((0, Np - N), (0, Np - N)))
    V = np.eye(Np)
    tiny = max(N * EPS * np.linalg.norm(A), 1e-300)
    for sweep in range(60):
        rot = False
        for r in range(Np - 1):
            J = np.eye(Np)
            for p, q in pairs(Np, r):
                apq, app, aqq = A[p, q], A[p, p], A[q, q]
                if apq * apq > EPS * EPS * abs(app * aqq) and abs(apq) > tiny:
                    d, tw = aqq - app, 2 * apq
                    t = np.copysign(1.0, d) * tw / (abs(d) + np.sqrt(d * d + tw * tw))
                    c = 1 / np.sqrt(1 + t * t)
                    s = t * c
                    J[p, p] = J[q, q] = c
                    J[p, q], J[q, p] = s, -s
                    rot = True
            A = J.T @ A @ J
            V = V @ J
        if not rot:
            return sweep + 1, V[:N, :N]
    return 60, V[:N, :N]


name = sys.argv[1] if len(sys.argv) > 1 else "pop6"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
prob = make_config(name)
o = HsdeOracle.from_problem(prob)
st = o.initial_state()
N = prob.psd_dims[0]
L = N * (N + 1) // 2
Vp = None
cold, warm = [], []
for k in range(iters):
    u1, u2, u3 = o.affine(st.xi + st.z, st.y + st.s, st.tau + st.kappa)
    a = (u1 - st.z)[o.n_free:o.n_free + L]
    A = smat(a, N)
    sc, V = jacobi(A)
    cold.append(sc)
    if Vp is not None:
        sw, Vb = jacobi(Vp.T @ A @ Vp)
        warm.append(sw)
        Vp = Vp @ Vb
    else:
        Vp = V
    st = o.step(st)
print(name, "N", N, "cold sweeps mean", np.mean(cold), "warm mean", np.mean(warm) if warm else None)
print("cold", cold)
print("warm", warm)
