"""In-graph (warm, concurrent) kernel durations per kernel name through CUPTI (torch.profiler):
python tools/kernel_times.py pop20 [iters] [skip]. The solver runs `skip` iterations first, then
`iters` profiled graph replays; the table is per iteration."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1708_04174_b200 import SosAdmm  # noqa: E402
from sosgen import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "pop20"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 50
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 200
g = SosAdmm.from_problem(make_config(cfg), tol=1e-300, max_iters=10 ** 9)
g.iterate(skip)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    g.iterate(iters)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
t0, t1 = None, None
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    name = e.name.split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    s, d = e.time_range.start, e.time_range.end
    t0 = s if t0 is None else min(t0, s)
    t1 = d if t1 is None else max(t1, d)
tot = sum(a[1] for a in agg.values())
print(f"{cfg}: {iters} iterations after {skip}; span {(t1 - t0) / iters:.1f} us / iteration, "
      f"kernel sum {tot / iters:.1f} us / iteration")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k[:48]:48s} {n / iters:6.1f} launches {t / iters:9.1f} us/it {t / n:8.2f} us/launch {100 * t / tot:5.1f}%")
