"""Probe: GPU trajectory (tau, residuals, pobj) every `stride` iterations, for comparison with the oracle's."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_04174_b200 import SosAdmm
from sosgen import make_config
name, kmax, stride = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
s = SosAdmm.from_problem(make_config(name), tol=1e-300, max_iters=1 << 40)
out = []
for k in range(stride, kmax + 1, stride):
    info = s.iterate(stride)
    out.append([info["iter"], info["tau"], info["res_pri"], info["res_dual"], info["res_gap"], info["pobj"]])
json.dump(out, open(f"gpurun_out/traj_{name}.json", "w"))
s2 = SosAdmm.from_problem(make_config(name), tol=1e-4, max_iters=20000)
print(name, "solver stop", s2.iterate(20000))
