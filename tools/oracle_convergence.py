"""Write the oracle's converged result for a BASELINE.json config to tests/golden/ (BJ acceptance:
converged objective within 1e-6 of the oracle's, iteration counts within 2%).

Calls only `oracle/` (and the seeded input generators of `sosgen/`): the stored values never come
from the CUDA path.  Single BLAS thread; the history is kept so that the gamma-accuracy iteration
(first k with max residual <= tol and |gamma / gamma0 - 1| <= 1e-4) is recorded too.

usage: OPENBLAS_NUM_THREADS=1 python tools/oracle_convergence.py pop40 [--tol 1e-4] [--max-iters 20000]
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import HsdeOracle, Status  # noqa: E402
from sosgen import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--tol", type=float, default=1e-4)
    ap.add_argument("--max-iters", type=int, default=20000)
    a = ap.parse_args()
    prob = make_config(a.name)
    t0 = time.time()
    orc = HsdeOracle.from_problem(prob)
    st, status, hist = orc.solve(tol=a.tol, max_iters=a.max_iters)
    g0 = prob.meta.get("gamma0")
    gacc = None
    if g0 is not None:
        for k, h in enumerate(hist, start=1):
            if max(h[0], h[1], h[2]) <= a.tol and abs(-h[3] / g0 - 1.0) <= 1e-4:
                gacc = k
                break
    rev = subprocess.run(["git", "-C", ROOT, "log", "-1", "--format=%h", "--", "oracle"], capture_output=True,
                         text=True).stdout.strip()
    out = dict(source=f"tools/oracle_convergence.py {a.name} --tol {a.tol} --max-iters {a.max_iters} "
                      f"(oracle/ at {rev}; plain FP64 CPU HSDE-ADMM, reading C9 stop rule)",
               config=a.name, seed=prob.meta.get("seed"), tol=a.tol, max_iters=a.max_iters,
               status=int(status), status_name=Status(status).name, iters=int(st.k),
               pobj=float(hist[-1][3]), res=[float(x) for x in hist[-1][:3]], tau=float(st.tau),
               kappa=float(st.kappa), gamma0=g0, gamma_acc_iter=gacc, cpu_seconds=time.time() - t0)
    path = os.path.join(ROOT, "tests", "golden", f"oracle_convergence_{a.name}.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
