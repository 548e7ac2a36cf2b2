"""Plain FP64 HSDE-ADMM (oracle; TEST INFRASTRUCTURE ONLY).

Follows PAPER.md §IV in the paper's order and notation, with no partial-orthogonality
shortcut (BASELINE.json `north_star`: "a dense or sparse LDL^T of
[I A^T; A -I], with no partial-orthogonality shortcut, and a LAPACK-style eigh"):

* HSDE: u = (xi, y, tau), v = (z, s, kappa), Q = [[0, -A^T, c], [A, 0, -b], [-c^T, b^T, 0]];
  cones C = K x R^m x R_+ and C* = K* x {0}^m x R_+, K = R^t x S_+ x ....
* ADMM (`eq:ADMMSteps`):
      u_hat = (I + Q)^{-1} (u + v);   u = P_C(u_hat - v);   v = v - u_hat + u.
* Linear step: with M = [[I, -A^T], [A, I]], zeta = (c, -b),
      [u_hat_1; u_hat_2] = [I - (M^{-1} zeta) zeta^T / (1 + zeta^T M^{-1} zeta)] M^{-1} [w1 - c w3; w2 + b w3],
      u_hat_3 = w3 + c^T u_hat_1 - b^T u_hat_2   (`E:FirstBlockElimination`).
  M^{-1} r is computed from ONE generic sparse LU of the quasi-definite KKT = [[I, A^T], [A, -I]]
  (SuperLU, symmetric mode, minimum-degree ordering on A^T + A, no pivoting: an LDL^T up to
  diagonal scaling): M [p1; p2] = r  <=>  KKT [p1; -p2] = r.
* The linear step is then refined (reading C15): two steps of iterative refinement on the
  HSDE system (I + Q) u_hat = omega itself with residuals in extended precision
  (np.longdouble), because the rank-one elimination loses up to ~1e-11 absolute in u_hat_3 when
  1 + zeta^T M^{-1} zeta is large (4e5 on pop20) and tau << 1.  The refined u_hat is the solution of
  the paper's linear system to working accuracy; the formula itself is unchanged.
* Residuals / termination: DESIGN.md reading C9 (corrected infeasibility tests).
* Initialisation: DESIGN.md reading C7: u0 = (0, 0, 1), v0 = (0, 0, 0).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from .psd import proj_psd_svec


class Status(enum.IntEnum):
    """Same codes as include/sosadmm.h `sosadmm_status`."""

    RUNNING = 0
    OPTIMAL = 1
    PRIMAL_INFEASIBLE = 2
    DUAL_INFEASIBLE = 3
    MAX_ITERS = 4
    INCONCLUSIVE = 5


@dataclass
class OracleState:
    xi: np.ndarray
    y: np.ndarray
    tau: float
    z: np.ndarray
    s: np.ndarray
    kappa: float
    k: int = 0

    def copy(self) -> "OracleState":
        return OracleState(self.xi.copy(), self.y.copy(), float(self.tau), self.z.copy(), self.s.copy(),
                           float(self.kappa), self.k)

    def u(self) -> np.ndarray:
        return np.concatenate([self.xi, self.y, [self.tau]])

    def v(self) -> np.ndarray:
        return np.concatenate([self.z, self.s, [self.kappa]])


@dataclass
class Residuals:
    pres: float
    dres: float
    gap: float
    pobj: float
    dobj: float
    pinf: float  # ||A^T y + z|| / (b^T y)   (inf if b^T y <= 0)
    dinf: float  # ||A xi|| / (-c^T xi)     (inf if c^T xi >= 0)
    extra: dict = field(default_factory=dict)


class HsdeOracle:
    def __init__(self, A, b, c, n_free: int, psd_dims: list[int], refine: int = 2):
        self.refine = int(refine)
        self.A = sp.csc_matrix(A, dtype=np.float64)
        self.m, self.n = self.A.shape
        self.b = np.asarray(b, dtype=np.float64)
        self.c = np.asarray(c, dtype=np.float64)
        self.n_free = int(n_free)
        self.psd_dims = [int(d) for d in psd_dims]
        assert self.n == self.n_free + sum(d * (d + 1) // 2 for d in self.psd_dims)
        KKT = sp.bmat([[sp.identity(self.n), self.A.T], [self.A, -sp.identity(self.m)]], format="csc")
        self.lu = splu(KKT, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                       options=dict(SymmetricMode=True))
        self.zeta = np.concatenate([self.c, -self.b])
        self.h = self.solve_M(self.zeta)            # M^{-1} zeta, cached
        self.denom = 1.0 + self.zeta @ self.h       # 1 + zeta^T M^{-1} zeta
        self.nb = np.linalg.norm(self.b)
        self.nc = np.linalg.norm(self.c)
        LD = np.longdouble
        self._A_ld = self.A.tocsr().astype(LD)
        self._AT_ld = self.A.T.tocsr().astype(LD)
        self._b_ld = self.b.astype(LD)
        self._c_ld = self.c.astype(LD)

    @staticmethod
    def from_problem(prob) -> "HsdeOracle":
        return HsdeOracle(prob.A, prob.b, prob.c, prob.n_free, prob.psd_dims)

    # ---------------------------------------------------------------- linear step
    def solve_M(self, r: np.ndarray) -> np.ndarray:
        """M^{-1} r with M = [[I, -A^T], [A, I]] via the KKT factorisation."""
        sol = self.lu.solve(np.asarray(r, dtype=np.float64))
        return np.concatenate([sol[:self.n], -sol[self.n:]])

    def affine(self, w1: np.ndarray, w2: np.ndarray, w3: float):
        """u_hat = (I + Q)^{-1} (w1, w2, w3), refined (reading C15)."""
        u1, u2, u3 = self.affine_once(w1, w2, w3)
        if self.refine <= 0:
            return u1, u2, u3
        LD = np.longdouble
        u1, u2, u3 = u1.astype(LD), u2.astype(LD), LD(u3)
        w1l, w2l, w3l = np.asarray(w1, dtype=LD), np.asarray(w2, dtype=LD), LD(w3)
        for _ in range(self.refine):
            # residual of (I + Q) u = w, Q of eq:DefinitionQ, in extended precision
            r1 = w1l - (u1 - self._AT_ld @ u2 + self._c_ld * u3)
            r2 = w2l - (self._A_ld @ u1 + u2 - self._b_ld * u3)
            r3 = w3l - (-(self._c_ld @ u1) + self._b_ld @ u2 + u3)
            d1, d2, d3 = self.affine_once(r1.astype(np.float64), r2.astype(np.float64), float(r3))
            u1, u2, u3 = u1 + d1, u2 + d2, u3 + LD(d3)
        return u1.astype(np.float64), u2.astype(np.float64), float(u3)

    def affine_once(self, w1: np.ndarray, w2: np.ndarray, w3: float):
        """One pass of `E:MatrixInverseResult` + `E:FirstBlockElimination`."""
        r = np.concatenate([w1 - self.c * w3, w2 + self.b * w3])
        p = self.solve_M(r)
        coef = (self.zeta @ p) / self.denom
        u12 = p - coef * self.h
        u1, u2 = u12[:self.n], u12[self.n:]
        u3 = w3 + self.c @ u1 - self.b @ u2
        return u1, u2, u3

    # ---------------------------------------------------------------- cone step
    def project_K(self, x: np.ndarray) -> np.ndarray:
        """P_K for K = R^t x S_+(N_1) x ...: free part unchanged, per-block eig clamp."""
        out = x.copy()
        off = self.n_free
        for N in self.psd_dims:
            L = N * (N + 1) // 2
            out[off:off + L] = proj_psd_svec(x[off:off + L], N)
            off += L
        return out

    # ---------------------------------------------------------------- iteration
    def initial_state(self) -> OracleState:
        """DESIGN.md reading C7: u0 = (0, 0, tau = 1), v0 = 0."""
        return OracleState(np.zeros(self.n), np.zeros(self.m), 1.0, np.zeros(self.n), np.zeros(self.m), 0.0, 0)

    def step(self, st: OracleState) -> OracleState:
        """One iteration of `eq:ADMMSteps`."""
        # eq:HsdeStep1: u_hat = (I + Q)^{-1} (u + v)
        u1, u2, u3 = self.affine(st.xi + st.z, st.y + st.s, st.tau + st.kappa)
        # eq:HsdeStep2: u = P_C(u_hat - v), C = K x R^m x R_+
        xi = self.project_K(u1 - st.z)
        y = u2 - st.s
        tau = max(0.0, u3 - st.kappa)
        # eq:HsdeStep3: v = v - u_hat + u
        z = st.z - u1 + xi
        s = st.s - u2 + y
        kappa = st.kappa - u3 + tau
        return OracleState(xi, y, tau, z, s, kappa, st.k + 1)

    # ---------------------------------------------------------------- residuals
    def residuals(self, st: OracleState) -> Residuals:
        """DESIGN.md reading C9, evaluated at (u^k, v^k)."""
        Ax = self.A @ st.xi
        ATy_z = self.A.T @ st.y + st.z
        cx = self.c @ st.xi
        by = self.b @ st.y
        pinf = np.linalg.norm(ATy_z) / by if by > 0 else np.inf
        dinf = np.linalg.norm(Ax) / (-cx) if cx < 0 else np.inf
        if st.tau <= 0.0:
            return Residuals(np.inf, np.inf, np.inf, np.nan, np.nan, pinf, dinf)
        t = st.tau
        pres = np.linalg.norm(Ax / t - self.b) / (1.0 + self.nb)
        dres = np.linalg.norm(ATy_z / t - self.c) / (1.0 + self.nc)
        pobj, dobj = cx / t, by / t
        gap = abs(pobj - dobj) / (1.0 + abs(pobj) + abs(dobj))
        return Residuals(pres, dres, gap, pobj, dobj, pinf, dinf)

    @staticmethod
    def classify(res: Residuals, tol: float) -> Status:
        """Termination rule (C9): Optimal first, then the two certificate tests."""
        if max(res.pres, res.dres, res.gap) <= tol:
            return Status.OPTIMAL
        if res.pinf <= tol:
            return Status.PRIMAL_INFEASIBLE
        if res.dinf <= tol:
            return Status.DUAL_INFEASIBLE
        return Status.RUNNING

    def solve(self, tol: float = 1e-4, max_iters: int = 2000, state: OracleState | None = None,
              callback=None, keep=0):
        """Iterate until the C9 rule fires or max_iters; returns (state, status, history).

        history[k-1] = (pres, dres, gap, pobj, tau, kappa) of iterate k; the first `keep`
        iterates are stored in history_states."""
        st = self.initial_state() if state is None else state.copy()
        hist, states = [], []
        status = Status.RUNNING
        while st.k < max_iters:
            st = self.step(st)
            if not (np.all(np.isfinite(st.xi)) and np.isfinite(st.tau)):
                raise FloatingPointError(f"non-finite iterate at k={st.k}")
            res = self.residuals(st)
            hist.append((res.pres, res.dres, res.gap, res.pobj, st.tau, st.kappa))
            if len(states) < keep:
                states.append(st.copy())
            if callback is not None:
                callback(st, res)
            status = self.classify(res, tol)
            if status != Status.RUNNING:
                break
        if status == Status.RUNNING:
            status = Status.MAX_ITERS
        self.history_states = states
        return st, status, hist
