"""GPU tests of the multi-GPU block-sharded mode (sosadmm_setup_sharded) at world
size 1 — this round runs on one GPU; the host orchestration at world size 2 is covered on CPU by
tests/test_parallel_cpu.py.  The sharded code path (owned-column partial gather, NCCL allreduce of
the 2m + 3 partial sums, replicated Woodbury / HSDE scalars, owner-only projection) must give the
same iterates as the single-GPU path and as the oracle."""
import numpy as np
import pytest

from oracle import HsdeOracle
from sosgen import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture
def nccl_id():
    """A fresh NCCL unique id per test (an id initialises exactly one communicator)."""
    from paper_1708_04174_b200.sosadmm import nccl_unique_id

    return nccl_unique_id()


def _state(g):
    return np.concatenate([g["xi"], g["y"], [g["tau"]], g["z"], g["s"], [g["kappa"]]])


@pytest.mark.parametrize("name", ["pop6", "lyap10", "box24"])
def test_sharded_world1_matches_single_gpu_and_oracle(name, nccl_id):
    from paper_1708_04174_b200 import SosAdmm
    from paper_1708_04174_b200.parallel import block_owner

    prob = make_config(name)
    owner = block_owner(prob.psd_dims, 1)
    sh = SosAdmm.from_problem(prob, shard=(0, 1, nccl_id, owner))
    one = SosAdmm.from_problem(prob)
    orc = HsdeOracle.from_problem(prob)
    st = orc.initial_state()
    worst = 0.0
    for k in range(1, 21):
        st = orc.step(st)
        ish = sh.iterate(1)
        ione = one.iterate(1)
        a, b = _state(sh.get_iterate()), _state(one.get_iterate())
        assert np.array_equal(a, b), (k, np.max(np.abs(a - b)))  # same arithmetic, bit-identical
        for key in ("tau", "kappa", "iter", "status"):
            assert ish[key] == ione[key]
        ref = np.concatenate([st.u(), st.v()])
        worst = max(worst, np.linalg.norm(a - ref) / np.linalg.norm(ref))
    assert worst <= 1e-9, worst
    # residuals: only the summation order of the orthogonal dual-residual partials differs
    for key in ("res_pri", "res_dual", "res_gap", "pobj"):
        assert abs(ish[key] - ione[key]) <= 1e-12 * max(1.0, abs(ione[key])), key
    with pytest.raises(RuntimeError):
        sh.project_psd(0, np.zeros(prob.psd_dims[0] * (prob.psd_dims[0] + 1) // 2))
    sh.close()
    one.close()


def test_sharded_rejects_bad_owner(nccl_id):
    from paper_1708_04174_b200 import SosAdmm

    prob = make_config("pop6")
    with pytest.raises(RuntimeError):
        SosAdmm.from_problem(prob, shard=(0, 1, nccl_id, np.array([3], dtype=np.int32)))


@pytest.mark.parametrize("peer", [False, True], ids=["devsum", "peer"])
@pytest.mark.parametrize("name,world,owner", [("lyap10", 2, [1, 0]), ("lyap10", 2, [0, 1]), ("box24", 2, None),
                                              ("box24", 4, None), ("box24", 8, None)])
def test_sharded_world_n_emulated(name, world, owner, peer):
    """The world >= 2 arithmetic (owned-column partial gathers k_gather_part / k_lowdual_part /
    k_shard_scalars, the 2m + 3 sum, replicated m-phase, owner-only projection) on one GPU:
    every rank's context on the same device, the partial sums added by a device kernel where the product
    path calls ncclAllReduce (NCCL refuses two ranks on one GPU).  20 iterates against the single-GPU path
    (1e-12: only the summation order of the partial sums differs) and the oracle (1e-9, reading C13).
    peer: the f4 path — each rank's k_gather_fin_peer reads every rank's partial buffer after the
    per-round flag hand-off (k_peer_signal) and adds them in rank order, fused into the gather's consumer;
    it must be bit-identical to the device-sum emulation (same rank-order sum)."""
    from paper_1708_04174_b200 import SosAdmm
    from paper_1708_04174_b200.parallel import block_owner
    from paper_1708_04174_b200.sosadmm import group_get_iterate, group_iterate, group_link_peers

    prob = make_config(name)
    own = np.array(owner if owner is not None else block_owner(prob.psd_dims, world), dtype=np.int32)
    assert len(set(own.tolist())) == min(world, len(prob.psd_dims))  # every rank that can own a block does
    ranks = [SosAdmm.from_problem(prob, shard=(r, world, None, own)) for r in range(world)]
    ref_ranks = None
    if peer:
        group_link_peers(ranks)
        ref_ranks = [SosAdmm.from_problem(prob, shard=(r, world, None, own)) for r in range(world)]
    one = SosAdmm.from_problem(prob)
    orc = HsdeOracle.from_problem(prob)
    st = orc.initial_state()
    worst_one = worst_orc = 0.0
    try:
        for k in range(1, 21):
            st = orc.step(st)
            group_iterate(ranks, 1)
            one.iterate(1)
            g = group_get_iterate(ranks)
            assert g["iter"] == k
            if ref_ranks is not None:  # peer reduction == device-sum emulation, bit for bit
                group_iterate(ref_ranks, 1)
                assert np.array_equal(_state(g), _state(group_get_iterate(ref_ranks))), k
            a, b = _state(g), _state(one.get_iterate())
            ref = np.concatenate([st.u(), st.v()])
            worst_one = max(worst_one, np.linalg.norm(a - b) / np.linalg.norm(b))
            worst_orc = max(worst_orc, np.linalg.norm(a - ref) / np.linalg.norm(ref))
    finally:
        for r in ranks + (ref_ranks or []):
            r.close()
        one.close()
    assert worst_one <= 1e-12, worst_one
    assert worst_orc <= 1e-9, worst_orc
