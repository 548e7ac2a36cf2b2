"""Probe: where the fixed cost of a solve goes (setup, first iterate = graph capture + module load,
steady iterations), for two problems in one process."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_04174_b200 import SosAdmm
from sosgen import ball_pop, make_config
for name, prob in [("ball10", ball_pop(10)), ("ball12", ball_pop(12)), ("ball10b", ball_pop(10)), ("pop20", make_config("pop20"))]:
    t0 = time.perf_counter(); s = SosAdmm.from_problem(prob, tol=1e-12, max_iters=100000)
    t1 = time.perf_counter(); s.iterate(1)
    t2 = time.perf_counter(); s.iterate(1)
    t3 = time.perf_counter(); s.iterate(50)
    t4 = time.perf_counter(); s.close()
    print(f"{name}: setup {1e3*(t1-t0):.1f} ms, first iterate(1) {1e3*(t2-t1):.1f} ms, second {1e3*(t3-t2):.2f} ms, 50 iters {1e3*(t4-t3):.2f} ms", flush=True)
