"""Host-side logic of the multi-GPU block sharding (paper_1708_04174_b200/parallel.py), on CPU with
the gloo backend at world size 2 (the GPU collective itself is exercised by
tests/test_gpu_sharded.py at world size 1 — one GPU per round)."""
import os
import socket

import numpy as np
import pytest

from paper_1708_04174_b200.parallel import assemble, block_owner, broadcast_id, owned_columns


def test_block_owner_lpt():
    dims = [325] + [25] * 24  # config 3: one sigma_0 Gram + 24 multiplier Grams
    for world in (1, 2, 4, 8):
        own = block_owner(dims, world)
        assert own.shape == (25,) and own.min() >= 0 and own.max() < world
        loads = np.zeros(world)
        for b, d in enumerate(dims):
            loads[own[b]] += float(d) ** 3
        # LPT: no rank exceeds the ideal share by more than the largest block
        assert loads.max() <= loads.sum() / world + 325.0 ** 3 + 1e-9
        assert np.array_equal(own, block_owner(dims, world))  # deterministic
    assert list(block_owner([65, 285], 2)) == [1, 0]
    assert list(block_owner([861], 8)) == [0]
    with pytest.raises(ValueError):
        block_owner([3], 0)


def test_owned_columns_partition():
    dims, nf = [3, 2, 4], 5
    own = block_owner(dims, 2)
    masks = [owned_columns(nf, dims, own, r) for r in range(2)]
    total = masks[0].astype(int) + masks[1].astype(int)
    assert np.all(total == 1)  # every column has exactly one authoritative rank
    assert masks[0][:nf].all() and not masks[1][:nf].any()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, nf = [65, 285], 1000  # config 2 (lyap10) shape
        own = block_owner(dims, world)
        nid = broadcast_id(bytes(range(128)) if rank == 0 else None)
        n = nf + sum(d * (d + 1) // 2 for d in dims)
        rng = np.random.default_rng(7)  # the same "true" iterate on every rank
        full = rng.standard_normal(n)
        mask = owned_columns(nf, dims, own, rank)
        local = np.where(mask, full, np.nan)  # non-owned entries are stale garbage on this rank
        got = assemble(np.nan_to_num(local, nan=1e300), mask)
        q.put((rank, list(own), nid == bytes(range(128)), float(np.max(np.abs(got - full)))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_orchestration():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][1] == res[1][1]  # identical block ownership on both ranks
    assert all(r[2] for r in res)  # the NCCL id reached every rank intact
    assert all(r[3] == 0.0 for r in res)  # exact assembly of the owned entries
