"""Probe: cost of the L2 flush on a small config's timed step (pop6) — per-step device time after a
512 MB write-flush, after a 512 MB read-flush, and with no flush; plus a trivial kernel as control."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1708_04174_b200 import SosAdmm
from sosgen import make_config

s = SosAdmm.from_problem(make_config(sys.argv[1] if len(sys.argv) > 1 else "pop6"), tol=1e-300, max_iters=1 << 40)
st = s.stream
buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
small = torch.zeros(1024, device="cuda")
s.iterate(300)
torch.cuda.synchronize()
def run(mode, what, K=100):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for i in range(K):
        with torch.cuda.stream(st):
            if mode == "write": buf.fill_(float(i))
            elif mode == "read": small[0] += buf.sum()
            elif mode == "write+small": buf.fill_(float(i)); small.add_(1.0)
            evs[i][0].record(st)
        if what == "iter": s.iterate_async(1)
        else:
            with torch.cuda.stream(st): small.add_(1.0)
        with torch.cuda.stream(st): evs[i][1].record(st)
    torch.cuda.synchronize()
    return 1e3 * sum(a.elapsed_time(b) for a, b in evs) / K
for what in ["iter", "trivial"]:
    for mode in ["none", "write", "read", "write+small"]:
        print(f"{what:8s} after {mode:12s}: {run(mode, what):8.1f} us/step", flush=True)
