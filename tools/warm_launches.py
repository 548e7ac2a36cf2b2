"""Launch list of warm-mode iterations for ncu (--profile-from-start off): advances a solve of the
config by `start` iterations un-profiled, then profiles `k` graph replays (cudaProfilerStart/Stop).
  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/warm_launches.py pop40 2000 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1708_04174_b200 import SosAdmm  # noqa: E402
from sosgen import make_config  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "pop40"
start = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 3
g = SosAdmm.from_problem(make_config(name), tol=1e-300, max_iters=1 << 40)
g.iterate(start)
torch.cuda.synchronize()
torch.cuda.profiler.start()
g.iterate_profiled(k)  # un-graphed launches (ncu does not descend into the graph IF nodes)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(g.warm_stats())
