"""Table I / Table II of the paper on one B200: solve the SDP relaxation of `eq:ExamplePOP`
(ball-constrained quartic POP, Lasserre order 2d = 4, weighted form with one multiplier)
with the CUDA path at the paper's tolerance, for every n of Table I.

Prints one JSON line per n: the sizes (checked against Table I), setup and iteration wall time,
iterations, status, gamma = -pobj, and Table II's objective values beside it.  The paper's
times are CPU (i7 2.8 GHz, MATLAB): context only, not a target.

usage: python tools/table1_gpu.py [--n 10 12 ...] [--tol 1e-3] [--max-iters 20000] [--out FILE]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1708_04174_b200 import SosAdmm  # noqa: E402
from sosgen import ball_pop  # noqa: E402

# Table I: N, m, t, CDCS-sos seconds (tol 1e-3); Table II:
# (interior point, SCS-direct, SCS-indirect, CDCS-sos); None = "**" (out of memory).
TABLE = {
    10: (66, 1000, 66, 0.4, (-9.11, -9.12, -9.13, -9.10)),
    12: (91, 1819, 91, 0.7, (-11.12, -11.10, -11.10, -11.11)),
    14: (120, 3059, 120, 1.4, (-13.12, -13.09, -13.09, -13.12)),
    17: (171, 5984, 171, 3.5, (-16.12, -16.09, -16.09, -16.06)),
    20: (231, 10625, 231, 8.5, (-19.12, -19.17, -19.17, -19.08)),
    24: (325, 20474, 325, 22.8, (-23.12, -23.04, -23.04, -23.15)),
    29: (465, 40919, 465, 67.1, (None, -28.17, -28.18, -28.17)),
    35: (666, 82250, 666, 216.9, (None, -34.05, -34.05, -34.08)),
    42: (946, 163184, 946, 686.6, (None, -41.21, -41.21, -41.05)),
}


def run(n, tol, max_iters):
    N, m_paper, t_paper, t_cdcs, objs = TABLE[n]
    t0 = time.perf_counter()
    prob = ball_pop(n)
    t1 = time.perf_counter()
    s = SosAdmm.from_problem(prob, tol=tol, max_iters=max_iters)
    s.iterate(0)
    t2 = time.perf_counter()
    info = s.iterate(max_iters)
    t3 = time.perf_counter()
    s.close()
    # our rows keep gamma's constant row: m = C(n+4,4) = Table I's m + 1 (reading on "-1")
    assert max(prob.psd_dims) == N and prob.m == m_paper + 1
    assert prob.psd_dims[0] * (prob.psd_dims[0] + 1) // 2 == t_paper  # multiplier svec = t
    gamma = -info["pobj"]
    ref = objs[0] if objs[0] is not None else float(np.mean(objs[1:]))
    return dict(n=n, N=N, m=prob.m, t_lowrank=t_paper + 1, tol=tol, status=info["status_name"],
                iters=info["iter"], gamma=gamma, rel_to_table2=abs(gamma - ref) / abs(ref),
                table2_ref=ref, table2_ref_kind="ipm" if objs[0] is not None else "mean of first-order",
                table2_row=objs, assemble_s=t1 - t0, setup_s=t2 - t1, solve_s=t3 - t2,
                ms_per_iter=1e3 * (t3 - t2) / max(info["iter"], 1), paper_cdcs_sos_s=t_cdcs,
                res=(info["res_pri"], info["res_dual"], info["res_gap"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="*", default=sorted(TABLE))
    ap.add_argument("--tol", type=float, default=1e-3)
    ap.add_argument("--max-iters", type=int, default=20000)
    ap.add_argument("--out")
    a = ap.parse_args()
    f = open(a.out, "w") if a.out else None
    for n in a.n:
        line = json.dumps(run(n, a.tol, a.max_iters))
        print(line, flush=True)
        if f:
            f.write(line + "\n")
            f.flush()


if __name__ == "__main__":
    main()
