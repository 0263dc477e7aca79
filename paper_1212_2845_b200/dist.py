"""Process-group plumbing for one-process-per-GPU runs (torch.distributed).

The data path never goes through torch: ghost planes move by NCCL send/recv
inside libvoxsim.so.  torch.distributed only bootstraps the library's NCCL
communicator (the 128-byte unique id) and reduces host-side timings.
"""
from __future__ import annotations

import os

from .lattice import nccl_unique_id, slab_planes


def env_ranks():
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def bootstrap_nccl_id(dist, rank):
    """Rank 0 creates the ncclUniqueId; every rank receives the same bytes."""
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def max_over_ranks(values, dist, device="cpu"):
    """Element-wise max of a list of floats over all ranks."""
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu()]


def gather_rows(values, dist, device="cpu"):
    """Every rank's list of floats, as a list of rows (rank order), on every rank."""
    import torch
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [[float(x) for x in t.cpu()]]
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [[float(x) for x in o.cpu()] for o in out]


def sum_over_ranks_u64(value, dist, device="cpu"):
    """Sum of a uint64 over all ranks, modulo 2^64 (a partition-invariant digest)."""
    import torch
    v = int(value) & 0xFFFFFFFFFFFFFFFF
    t = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v], dtype=torch.int64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)   # two's-complement wraparound
    return int(t.cpu()[0]) & 0xFFFFFFFFFFFFFFFF


def ghost_planes(nx, nranks, rank):
    """(x0, x1, xl0, xl1): owned planes and the local box with its ghost planes,
    as libvoxsim lays out a rank's slab."""
    x0, x1 = slab_planes(nx, nranks, rank)
    return x0, x1, max(x0 - 1, 0), min(x1 + 1, nx)
