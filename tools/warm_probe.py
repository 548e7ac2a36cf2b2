"""Warm-started large-block projection on the GPU: iterates of the warm mode against the cold mode
(SOSADMM_WARM=0, a second process) and the oracle, the warm counters, and the graph-replay time per
iteration at several points of a solve.  Usage: python tools/warm_probe.py pop20 [iters]"""
import json
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(name, iters, chunk):
    import torch
    from paper_1708_04174_b200 import SosAdmm
    from sosgen import make_config

    prob = make_config(name)
    g = SosAdmm.from_problem(prob, tol=1e-300, max_iters=1 << 40)
    out = []
    done = 0
    while done < iters:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g.iterate(chunk)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        done += chunk
        it = g.get_iterate()
        ws = g.warm_stats()
        out.append({"k": done, "ms_per_iter": 1e3 * dt / chunk, "tau": it["tau"], "ws": ws,
                    "xi_norm": float(np.linalg.norm(it["xi"]))})
    it = g.get_iterate()
    return out, {k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in it.items()}


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        name, iters, chunk = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
        out, it = run(name, iters, chunk)
        print(json.dumps({"trace": out, "iterate": it}))
        sys.exit(0)
    name = sys.argv[1] if len(sys.argv) > 1 else "pop20"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    res = {}
    for mode in ["1", "0"]:
        env = dict(os.environ, SOSADMM_WARM=mode)
        p = subprocess.run([sys.executable, __file__, "--child", name, str(iters), str(chunk)], env=env,
                           capture_output=True, text=True, timeout=3000)
        if p.returncode != 0:
            print(p.stderr[-3000:])
            sys.exit(1)
        res[mode] = json.loads(p.stdout.strip().splitlines()[-1])
        for r in res[mode]["trace"]:
            print(f"warm={mode} k={r['k']:6d} {r['ms_per_iter']:.3f} ms/iter tau={r['tau']:.3e} ws={r['ws']}")
    a, b = res["1"]["iterate"], res["0"]["iterate"]
    u = lambda it: np.concatenate([it["xi"], it["y"], [it["tau"]], it["z"], it["s"], [it["kappa"]]])
    du = np.linalg.norm(u(a) - u(b)) / np.linalg.norm(u(b))
    print(f"{name}: after {iters} iterations warm vs cold relative difference {du:.3e}")
