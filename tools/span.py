"""Graph-replay time per iteration at one point of a solve (CUDA events, no profiler), for A/B runs of
environment switches: python tools/span.py pop40 2000 200 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1708_04174_b200 import SosAdmm  # noqa: E402
from sosgen import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "pop40"
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
g = SosAdmm.from_problem(make_config(cfg), tol=1e-300, max_iters=10 ** 9)
g.iterate(skip)
torch.cuda.synchronize()
out = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(g.stream)
    g.iterate_async(iters)
    b.record(g.stream)
    torch.cuda.synchronize()
    out.append(a.elapsed_time(b) * 1e3 / iters)
it = g.get_iterate()
print(f"{cfg} skip={skip} env={os.environ.get('TAG', '')} us/iter={' '.join(f'{v:.1f}' for v in out)} "
      f"warm={g.warm_stats()} tau={it['tau']:.6e}")
