import sys, numpy as np
sys.path.insert(0, '.')
from oracle import HsdeOracle
from sosgen import make_config
from paper_1708_04174_b200 import SosAdmm
for name in sys.argv[1:]:
    prob = make_config(name)
    gpu = SosAdmm.from_problem(prob); orc = HsdeOracle.from_problem(prob)
    st = orc.initial_state()
    for k in range(1, 21):
        st = orc.step(st); gpu.iterate(1); g = gpu.get_iterate()
        scale = np.linalg.norm(np.concatenate([st.u(), st.v()]))
        du = np.linalg.norm(np.concatenate([g["xi"], g["y"], [g["tau"]]]) - st.u())/scale
        dv = np.linalg.norm(np.concatenate([g["z"], g["s"], [g["kappa"]]]) - st.v())/scale
        t = prob.n_free
        dxi = np.linalg.norm(g["xi"][t:]-st.xi[t:])/scale; dz = np.linalg.norm(g["z"][t:]-st.z[t:])/scale
        dy = np.linalg.norm(g["y"]-st.y)/scale
        print(name, k, g["iter"], f"du={du:.2e} dv={dv:.2e} dxi={dxi:.2e} dz={dz:.2e} dy={dy:.2e} tau {g['tau']:.6e} {st.tau:.6e}", flush=True)
