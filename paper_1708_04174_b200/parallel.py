"""Multi-GPU block sharding: host-side orchestration of `sosadmm_setup_sharded`.

One process per GPU (torchrun).  The PSD blocks of ONE program are partitioned over the ranks by
`block_owner` (longest-processing-time greedy on the per-block eigensolver cost, ~N^3, ties to the
lower rank, identical on every rank); rank 0 creates the NCCL unique id and `broadcast_id` sends it
over any torch.distributed process group (gloo or nccl).  Everything numeric happens inside the C
library: per iteration one ncclAllReduce of the length-m partial sums (include/sosadmm.h).
`assemble` is the host-side counterpart of the library's owned-entry allreduce, for callers that
hold per-rank copies (and for the CPU tests)."""
from __future__ import annotations

import numpy as np


def block_cost(N: int) -> float:
    """Relative cost of one PSD block per iteration: the N^3 eigensolver dominates."""
    return float(N) ** 3


def block_owner(psd_dims, world: int) -> np.ndarray:
    """Deterministic LPT assignment of the PSD blocks to `world` ranks (largest block first, to the
    currently least-loaded rank, ties to the lower rank)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    dims = [int(d) for d in psd_dims]
    order = sorted(range(len(dims)), key=lambda b: (-dims[b], b))
    load = [0.0] * world
    owner = np.zeros(len(dims), dtype=np.int32)
    for b in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[b] = r
        load[r] += block_cost(dims[b])
    return owner


def owned_columns(n_free: int, psd_dims, owner, rank: int) -> np.ndarray:
    """Column mask of the entries rank `rank` is authoritative for (free columns: rank 0)."""
    mask = np.zeros(n_free + sum(d * (d + 1) // 2 for d in psd_dims), dtype=bool)
    if rank == 0:
        mask[:n_free] = True
    col = n_free
    for b, d in enumerate(psd_dims):
        L = d * (d + 1) // 2
        if owner[b] == rank:
            mask[col:col + L] = True
        col += L
    return mask


def broadcast_id(nccl_id: bytes | None, group=None) -> bytes:
    """Broadcast rank 0's NCCL unique id (128 bytes) to every rank of a torch.distributed group."""
    import torch.distributed as dist

    obj = [nccl_id if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != 128:
        raise RuntimeError("NCCL unique id broadcast failed")
    return bytes(obj[0])


def assemble(local: np.ndarray, mask: np.ndarray, group=None) -> np.ndarray:
    """Full column vector from per-rank copies whose authoritative entries are `mask` (sum of the
    masked copies over the ranks; exact since every entry has exactly one owner)."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.where(mask, local, 0.0).astype(np.float64))
    dist.all_reduce(t, group=group)
    return t.numpy()


def sharded_solver(prob, rank: int, world: int, device: int, group=None, **kw):
    """Construct the rank's `SosAdmm` of a block-sharded solve (collective over `group`)."""
    from .sosadmm import SosAdmm, nccl_unique_id

    owner = block_owner(prob.psd_dims, world)
    nid = broadcast_id(nccl_unique_id() if rank == 0 else None, group)
    return SosAdmm.from_problem(prob, device=device, shard=(rank, world, nid, owner), **kw), owner
