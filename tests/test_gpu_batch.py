"""batched independent instances on one GPU (sosadmm_iterate_async + iterate_batch).

Each instance owns a stream and its own CUDA graph; iterate_batch enqueues every instance's graph
replays before waiting, so the instances run concurrently.  The arithmetic of an instance does not
depend on what runs beside it (fixed-order reductions, no shared state), so every batched iterate
must be BIT-identical to the same instance run alone, and each instance must stop at its own
residual-stop iteration.  Per-instance parity with the oracle is covered by test_gpu_parity.py.
"""
import numpy as np
import pytest

from sosgen import make_config

pytestmark = pytest.mark.gpu


def _iterates(s):
    g = s.get_iterate()
    return np.concatenate([g["xi"], g["y"], g["z"], g["s"], [g["tau"], g["kappa"], g["iter"]]])


def _solo_and_batch(probs, k, chunk=256, **kw):
    from paper_1708_04174_b200 import SosAdmm, iterate_batch

    solo = []
    for p in probs:
        s = SosAdmm.from_problem(p, **kw)
        info = s.iterate(k)
        solo.append((info, _iterates(s)))
        s.close()
    batch = [SosAdmm.from_problem(p, **kw) for p in probs]
    infos = iterate_batch(batch, k, chunk=chunk)
    out = [(infos[i], _iterates(b)) for i, b in enumerate(batch)]
    for b in batch:
        b.close()
    return solo, out


@pytest.mark.parametrize("names", [[("pop6", 0), ("pop6", 1), ("pop6", 2)],
                                   [("pop20", 0), ("lyap10", 0), ("pop6", 3), ("pop20", 1)]])
def test_batch_bit_identical_to_solo(names):
    probs = [make_config(n, seed=s) for n, s in names]
    solo, batch = _solo_and_batch(probs, 20, max_iters=10_000)
    for (si, sv), (bi, bv) in zip(solo, batch):
        assert bi["iter"] == si["iter"] == 20
        assert np.array_equal(sv, bv)
        assert bi["res_pri"] == si["res_pri"] and bi["res_dual"] == si["res_dual"]


@pytest.mark.parametrize("chunk", [256, 7])
def test_batch_independent_termination(chunk):
    """Instances converge at different iterations; each stops at its own residual-stop k (whatever the
    enqueue round size, finished instances drop out between rounds)."""
    probs = [make_config("pop6", seed=s) for s in range(4)]
    solo, batch = _solo_and_batch(probs, 5000, chunk=chunk, max_iters=5000)
    its = [si["iter"] for si, _ in solo]
    assert len(set(its)) > 1  # the seeds really do stop at different iterations
    for (si, sv), (bi, bv) in zip(solo, batch):
        assert si["status_name"] == bi["status_name"] == "OPTIMAL"
        assert bi["iter"] == si["iter"]
        assert np.array_equal(sv, bv)


def test_get_iterate_into_preallocated_buffers():
    """get_iterate(out=...) (the e2e path copies into pinned host buffers) returns the same iterate."""
    from paper_1708_04174_b200 import SosAdmm

    s = SosAdmm.from_problem(make_config("pop6"))
    s.iterate(7)
    ref = s.get_iterate()
    out = {k: np.full_like(ref[k], np.nan) for k in ("xi", "y", "z", "s")}
    got = s.get_iterate(out=out)
    for k in ("xi", "y", "z", "s"):
        assert got[k] is out[k] and np.array_equal(out[k], ref[k])
    assert (got["tau"], got["kappa"], got["iter"]) == (ref["tau"], ref["kappa"], ref["iter"])
    with pytest.raises(ValueError):
        s.get_iterate(out={k: np.zeros(3) for k in ("xi", "y", "z", "s")})
    s.close()


def test_iterate_stops_enqueueing_after_termination():
    """iterate(k) with k far beyond the stop returns promptly (chunked enqueue with device-state polling)
    and leaves exactly the iterate of a run that asked for just a few more iterations than needed."""
    import time

    from paper_1708_04174_b200 import SosAdmm

    prob = make_config("pop6")
    s = SosAdmm.from_problem(prob, max_iters=10**7)
    s.iterate(1)
    t0 = time.perf_counter()
    info = s.iterate(10**7 - 1)
    dt = time.perf_counter() - t0
    assert info["status_name"] == "OPTIMAL" and dt < 5.0, dt
    r = SosAdmm.from_problem(prob, max_iters=10**7)
    ri = r.iterate(info["iter"] + 3)
    assert ri["iter"] == info["iter"]
    assert np.array_equal(_iterates(s), _iterates(r))
    s.close()
    r.close()


@pytest.mark.parametrize("name", ["pop6", "pop20"])
def test_fused_low_phase_bit_identical(name, monkeypatch):
    """For t' <= 16 k_tphase does k_lowT's and k_kinv's work itself (two launches less; the same warp
    sums).  The iterates must be BIT-identical to the three-launch chain (SOSADMM_NO_FUSE_LOW=1, read
    at setup), which test_gpu_parity.py checks against the oracle."""
    from paper_1708_04174_b200 import SosAdmm

    prob = make_config(name)
    out = []
    for env in (None, "1"):
        if env is None:
            monkeypatch.delenv("SOSADMM_NO_FUSE_LOW", raising=False)
        else:
            monkeypatch.setenv("SOSADMM_NO_FUSE_LOW", env)
        s = SosAdmm.from_problem(prob, max_iters=10_000)
        info = s.iterate(40)
        out.append((info, _iterates(s)))
        s.close()
    (ia, va), (ib, vb) = out
    assert ia["iter"] == ib["iter"] == 40
    assert np.array_equal(va, vb)
    assert ia["res_pri"] == ib["res_pri"] and ia["res_dual"] == ib["res_dual"]


def test_shared_gpu_hint_changes_no_iterate():
    """sosadmm_set_shared_gpu is a scheduling hint: with it the warm-start predictor of the large-block
    projection stays in line, without it the CUDA graph forks it beside the affine chain.  The predictor
    reads only what the previous iteration left, so the iterates are BIT-identical either way, also when the
    hint is flipped in the middle of a solve (the graph is rebuilt).  pop20: N = 231, predictor active."""
    from paper_1708_04174_b200 import SosAdmm

    prob = make_config("pop20")
    out = []
    for mode in ("lone", "shared", "flip"):
        s = SosAdmm.from_problem(prob, tol=1e-300, max_iters=1 << 30)
        if mode == "shared":
            s.set_shared_gpu(True)
        s.iterate(300)
        if mode == "flip":
            s.set_shared_gpu(True)
        info = s.iterate(300)
        ws = s.warm_stats()
        out.append((info, _iterates(s), ws))
        s.close()
    assert out[0][2][0]["warm"] > 400  # the refinement (and its predictor) carried the solve
    for info, v, _ in out[1:]:
        assert info["iter"] == out[0][0]["iter"] == 600
        assert np.array_equal(v, out[0][1])
