"""CPU FP64 oracle for the HSDE-ADMM hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import or execute anything under `oracle/`.  The product path
(`paper_1708_04174_b200`) never imports it and shares no code with it.

What it computes: the ADMM of PAPER.md `eq:ADMMSteps` on the
homogeneous self-dual embedding, with the linear step solved WITHOUT partial
orthogonality through a generic sparse LU of the quasi-definite KKT matrix [[I, A^T], [A, -I]]
(the "direct" method of P:881), the rank-one HSDE correction of `E:MatrixInverseResult`
(P:437-446), and the PSD projection by LAPACK `dsyevd` per block.

Pins (tests/test_oracle_*.py, `-m "not gpu"`), each independent of the oracle's own formulas:
* structure: brute-force ordered-pair enumeration of the indicator matrices B_alpha,
  Proposition 1 counts, sum_alpha n_alpha = N^2, n=1 d=1 -> D = diag(1, 2, 1);
* linear step: the materialised I + Q built from the HSDE definition times u-hat
  reproduces omega; dense LU of I + Q at tiny sizes; Q skew; denom >= 1;
* projection: diag(1, -2) -> diag(1, 0), idempotence, Moreau orthogonality, nonexpansiveness;
* whole iteration: the planted KKT point is an exact fixed point (closed form); the converged
  objective equals the planted optimum gamma0 = 1 (closed form); (x+1)^2 is feasible and
  -1-x^2 is certified infeasible;
* Table II of the paper: ball-constrained POP n = 10 optimum -9.11.
Iteration counts are "parity unpinned" by the paper (it prints none); see DESIGN.md.
"""
from .hsde_admm import HsdeOracle, OracleState, Status  # noqa: F401
from .psd import proj_psd_svec, smat, svec  # noqa: F401
from .structure import brute_force_structure  # noqa: F401
