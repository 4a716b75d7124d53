"""Sharded local orderings of one very large mesh (BASELINE configs[2] "C3",
SURVEY §8e).

Every rank holds the CSR and runs patching and the ND tree itself (the tree
is identical on every rank: the path is deterministic, so there is nothing
to broadcast).  The tree's subtrees at level k = ceil(log2 world) are dealt
to ranks by largest-first (LPT) on their vertex counts, the k top
separators likewise; each rank orders only its nodes (`mp_order_subtrees`)
and scatters their permutation entries.  In the postorder schedule a
subtree is a contiguous position range, so a rank's entries are a few
ranges; one all-gather of those ranges (NCCL on GPUs, gloo in the CPU tests)
is the path's only collective -- the "final permutation gather" of the
north star.

Reference: order_tree_nodes (local_order.cpp:77-86, its nodes are
independent) and compute_perm / schedule_postorder (assemble.cpp:24-85).
"""
from __future__ import annotations

import math

import numpy as np


def schedule(L: int, kind: str = "postorder") -> list[int]:
    """schedule_postorder / schedule_levelorder (assemble.cpp:24-46)."""
    nn = (1 << (L + 1)) - 1
    if kind == "levelorder":
        return [i for lev in range(L, -1, -1) for i in range((1 << lev) - 1, (1 << (lev + 1)) - 1)]
    out: list[int] = []

    def rec(i):
        if i >= nn:
            return
        rec(2 * i + 1)
        rec(2 * i + 2)
        out.append(i)
    rec(0)
    return out


def node_positions(node_offsets: np.ndarray, L: int, kind: str = "postorder") -> np.ndarray:
    """First permutation position of every node (compute_perm's running offset)."""
    nn = (1 << (L + 1)) - 1
    size = np.diff(np.asarray(node_offsets, np.int64))
    pos = np.zeros(nn + 1, np.int64)
    run = 0
    for i in schedule(L, kind):
        pos[i] = run
        run += int(size[i])
    pos[nn] = run
    return pos


def level_of(i: int) -> int:
    return (i + 1).bit_length() - 1


def owners(node_offsets: np.ndarray, L: int, world: int) -> np.ndarray:
    """Owning rank of every tree node.  Level-k subtrees (k = ceil(log2 world),
    capped at L) and then the top nodes are assigned largest-first to the
    least-loaded rank (ties: lower rank, then lower node id) -- deterministic
    from the tree alone, so every rank computes the same map."""
    nn = (1 << (L + 1)) - 1
    own = np.zeros(nn, np.int32)
    if world <= 1:
        return own
    size = np.diff(np.asarray(node_offsets, np.int64))
    k = min(L, math.ceil(math.log2(world)))
    roots = list(range((1 << k) - 1, (1 << (k + 1)) - 1))

    def subtree(r):
        out, st = [], [r]
        while st:
            i = st.pop()
            if i < nn:
                out.append(i)
                st += [2 * i + 1, 2 * i + 2]
        return out

    members = {r: subtree(r) for r in roots}
    weight = {r: int(size[members[r]].sum()) for r in roots}
    load = np.zeros(world, np.int64)
    for r in sorted(roots, key=lambda r: (-weight[r], r)):
        dst = int(np.argmin(load))
        own[members[r]] = dst
        load[dst] += weight[r]
    for i in sorted(range((1 << k) - 1), key=lambda i: (-int(size[i]), i)):
        dst = int(np.argmin(load))
        own[i] = dst
        load[dst] += int(size[i])
    return own


def rank_ranges(node_offsets: np.ndarray, L: int, own: np.ndarray, rank: int,
                kind: str = "postorder") -> list[tuple[int, int]]:
    """Merged (start, length) permutation ranges owned by `rank`, ascending."""
    pos = node_positions(node_offsets, L, kind)
    size = np.diff(np.asarray(node_offsets, np.int64))
    segs = sorted((int(pos[i]), int(size[i])) for i in np.nonzero(own == rank)[0] if size[i] > 0)
    out: list[tuple[int, int]] = []
    for s, n in segs:
        if out and out[-1][0] + out[-1][1] == s:
            out[-1] = (out[-1][0], out[-1][1] + n)
        else:
            out.append((s, n))
    return out


def gather_perm(perm, node_offsets, L, own, world, rank, kind="postorder"):
    """All-gather the owned permutation ranges of every rank into `perm` (a
    torch tensor, CUDA for NCCL or CPU for gloo) in place; returns it."""
    if world == 1:
        return perm
    import torch
    import torch.distributed as dist
    ranges = [rank_ranges(node_offsets, L, own, r, kind) for r in range(world)]
    counts = [sum(n for _, n in rr) for rr in ranges]
    width = max(counts)
    mine = [perm[s:s + n] for s, n in ranges[rank]]
    send = torch.zeros(width, dtype=perm.dtype, device=perm.device)
    if mine:
        send[:counts[rank]] = torch.cat(mine)
    recv = torch.empty(world * width, dtype=perm.dtype, device=perm.device)
    dist.all_gather_into_tensor(recv, send)
    for r in range(world):
        if r == rank:
            continue
        at = r * width
        for s, n in ranges[r]:
            perm[s:s + n] = recv[at:at + n]
            at += n
    return perm


def order_subtrees_device(ctx, n, offsets_ptr, neighbors_ptr, L, node_offsets_ptr, node_vertices_ptr,
                          mask_ptr, local_perm_ptr, perm_ptr, mode="approx_md", schedule_kind="postorder"):
    """mp_order_subtrees on device pointers."""
    import ctypes as C
    from ._lib import LOCAL_MODES, SCHEDULES, MpCsr, check, lib
    csr = MpCsr(n, C.c_void_p(offsets_ptr), C.c_void_p(neighbors_ptr), 1)
    check(lib().mp_order_subtrees(ctx.handle, C.byref(csr), L, C.c_void_p(node_offsets_ptr),
                                  C.c_void_p(node_vertices_ptr), LOCAL_MODES[mode], SCHEDULES[schedule_kind],
                                  C.c_void_p(mask_ptr), C.c_void_p(local_perm_ptr), C.c_void_p(perm_ptr), 1))
