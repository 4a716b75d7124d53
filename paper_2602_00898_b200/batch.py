"""Batches of independent meshes (BASELINE configs[3], SURVEY §8e "C4").

Frames shard across ranks with no data-path collective (each frame is ordered
entirely on one GPU); within a GPU several frames run concurrently, one
context (stream + workspace) per worker thread, because most stages of one
frame occupy only a few SMs.  Results can be gathered to rank 0 over
torch.distributed (NCCL on GPUs, gloo in the CPU tests) -- the only
collective, and off the timed path.
"""
from __future__ import annotations

import numpy as np


def shard(n_items: int, world: int, rank: int) -> list[int]:
    """Round-robin frame ids of `rank` (frame f -> rank f % world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return list(range(rank, n_items, world))


def owner(frame: int, world: int) -> int:
    return frame % world


class FramePool:
    """`workers` contexts on one device, driven by the native mp_order_batch
    (one library host thread per context)."""

    def __init__(self, device: int = 0, workers: int = 4):
        from .api import Context
        from ._lib import check, lib
        self.device = device
        self.ctx = [Context(device) for _ in range(workers)]
        for c in self.ctx:  # concurrent contexts: grid-wide kernels take 1/workers of the SMs each
            check(lib().mp_context_set_sm_share(c.handle, workers))

    def order_all(self, graphs, **kw):
        """Every graph ordered concurrently over the pool's contexts (host
        arrays in and out) through the native mp_order_batch."""
        from .api import order_batch
        return order_batch(graphs, self.ctx, **kw)

    def close(self):
        for c in self.ctx:
            c.close()


def gather_to_root(local: dict, world: int, rank: int):
    """Gather {frame: payload} dicts from every rank to rank 0 (None elsewhere)."""
    if world == 1:
        return dict(local)
    import torch.distributed as dist
    out = [None] * world if rank == 0 else None
    dist.gather_object(local, out, dst=0)
    if rank != 0:
        return None
    merged = {}
    for part in out:
        merged.update(part)
    return merged


def frame_digest(perm: np.ndarray, nnz_l: int) -> tuple:
    """Small per-frame payload for the gather (the full permutation stays local)."""
    import hashlib
    return (hashlib.sha256(np.ascontiguousarray(perm).tobytes()).hexdigest()[:16], int(nnz_l))


def max_over_ranks(x: float, world: int) -> float:
    """Max of a host scalar over the ranks (CPU tensor for gloo, CUDA for NCCL)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
