"""Short solves of every path (meant for compute-sanitizer: `compute-sanitizer --tool memcheck python
tools/sanitize.py [iters]`; compute-sanitizer is closed on this GPU pool, so here it only serves as a
plain all-paths smoke run: python tools/sanitize.py [iters]).
Covers the Jacobi path (pop6, N = 28), the large-block path with the cold eigensolver and the
warm-started refinement (pop12, N = 91 and a boxed POP with N = 66 + 11 small blocks), the t' > 1
Woodbury chain (lyap6, N = 27 + 83) and a batch of two instances; every run goes through the C ABI and the CUDA graph."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1708_04174_b200 import SosAdmm, iterate_batch  # noqa: E402
from sosgen import make_config  # noqa: E402
from sosgen.configs import lyapunov, planted_pop  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 30
probs = [make_config("pop6"), planted_pop("pop12", 12, 4, seed=2), planted_pop("box10", 10, 4, seed=3, box=True),
         lyapunov("lyap6", 6, seed=1)]
for p in probs:
    g = SosAdmm.from_problem(p, tol=1e-300, max_iters=1 << 30)
    info = g.iterate(k)
    torch.cuda.synchronize()
    ws = g.warm_stats() if hasattr(g, "warm_stats") else None
    print(p.name, p.psd_dims[:3], "iter", info["iter"], "res", info["res_pri"], info["res_dual"], "warm", ws, flush=True)
    g.close()
two = [SosAdmm.from_problem(make_config("pop6", seed=s), tol=1e-300, max_iters=1 << 30) for s in (0, 1)]
infos = iterate_batch(two, k)
print("batch", [i["iter"] for i in infos], flush=True)
for g in two:
    g.close()
print("sanitize run done")
