"""Per-evaluation trace of the warm refinement (coupling, orthonormality, Gershgorin bound at every S
evaluation of one ADMM iteration) at points along a solve.  Usage: python tools/warm_trace.py pop40 8000 500"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1708_04174_b200 import SosAdmm  # noqa: E402
from sosgen import make_config  # noqa: E402

WM_MAXS = 10


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "pop40"
    total = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
    every = int(sys.argv[3]) if len(sys.argv) > 3 else 500
    g = SosAdmm.from_problem(make_config(name), tol=1e-300, max_iters=1 << 40)
    L = g.lib
    L.sosadmm_debug_warm_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.sosadmm_debug_warm_trace.restype = ctypes.c_int
    out = np.zeros(4 * WM_MAXS + 8)
    done = 0
    first = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    while done < first:  # every iteration of the start of the solve
        g.iterate(1)
        done += 1
        show(L, g, out, done)
    while done < total:
        g.iterate(every - 5)
        done += every - 5
        for _ in range(5):
            g.iterate(1)
            done += 1
            show(L, g, out, done)


def show(L, g, out, done):
    rc = L.sosadmm_debug_warm_trace(g._ctx, 0, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0
    ne = int(out[3 * WM_MAXS])
    eta = " ".join(f"{v:.1e}" for v in out[:ne])
    rn = " ".join(f"{v:.1e}" for v in out[WM_MAXS:WM_MAXS + ne])
    gg = " ".join(f"{v:.1e}" for v in out[2 * WM_MAXS:2 * WM_MAXS + ne])
    ro = " ".join(f"{v:.1e}" for v in out[3 * WM_MAXS + 8:3 * WM_MAXS + 8 + ne])
    t = [int(v) for v in out[3 * WM_MAXS:3 * WM_MAXS + 8]]
    print(f"k={done:6d} evals={t[0]} cl0={t[1]} pred={t[2]} status={t[3]} why={t[4]} backoff={t[5]} fails={t[6]} "
          f"maxcl={t[7]} eta=[{eta}] rn=[{rn}] ro=[{ro}] g=[{gg}]", flush=True)


if __name__ == "__main__":
    main()
