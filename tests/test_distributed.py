"""CPU multi-process tests of the N>1 host logic (gloo, world size 2).

Frames (independent meshes, BASELINE configs[3]) shard round-robin across
ranks with no collective on the data path; results gather to rank 0.  The
per-frame ordering here is the CPU oracle (this is a test of the sharding and
gather logic, not of the kernels): the gathered result must equal the
single-process result for every frame, whatever the rank count.
"""
import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT

from paper_2602_00898_b200.batch import frame_digest, gather_to_root, max_over_ranks, owner, shard


def test_shard_is_a_balanced_partition():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            parts = [shard(n, world, r) for r in range(world)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
            assert all(owner(i, world) == r for r, p in enumerate(parts) for i in p)
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def _frames():
    import paper_2602_00898_b200 as mp
    return [mp.mesh_to_graph(mp.make_random_mesh(18 + f, 21, seed=f)) for f in range(5)]


def _order_frame(g):
    from oracle.oracle import Restatement
    R = Restatement()
    o = R.order(g, patch_size=24)
    return frame_digest(o["perm"], R.elimination_fill(g, o["perm"])["nnz_L"])


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    frames = _frames()
    local = {f: _order_frame(frames[f]) for f in shard(len(frames), world, rank)}
    merged = gather_to_root(local, world, rank)
    t = max_over_ranks(float(rank + 1), world)
    if rank == 0:
        q.put((merged, t))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_frames_match_single_process():
    import torch.multiprocessing as tmp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    merged, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    frames = _frames()
    expect = {f: _order_frame(frames[f]) for f in range(len(frames))}
    assert merged == expect
    assert tmax == 2.0


def test_subtree_owners_cover_and_balance():
    from paper_2602_00898_b200 import subtree as st
    rng = np.random.default_rng(3)
    L = 5
    nn = (1 << (L + 1)) - 1
    sizes = rng.integers(0, 50, nn)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    n = int(off[-1])
    for world in (1, 2, 3, 5, 8):
        own = st.owners(off, L, world)
        cover = np.zeros(n, np.int32)
        for r in range(world):
            for s, k in st.rank_ranges(off, L, own, r):
                cover[s:s + k] += 1
        assert np.all(cover == 1)
        # a subtree below level k is owned by one rank
        k = min(L, int(np.ceil(np.log2(world)))) if world > 1 else 0
        for i in range(nn):
            if (i + 1).bit_length() - 1 > k:
                assert own[i] == own[(i - 1) // 2]
    # postorder positions equal the schedule scan
    pos = st.node_positions(off, L)
    order = st.schedule(L)
    assert pos[order[0]] == 0 and pos[nn] == n


def _gather_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2602_00898_b200 import subtree as st
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    L = 4
    nn = (1 << (L + 1)) - 1
    sizes = np.random.default_rng(11).integers(0, 30, nn)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    n = int(off[-1])
    truth = np.random.default_rng(5).permutation(n).astype(np.int32)
    own = st.owners(off, L, world)
    perm = torch.full((n,), -1, dtype=torch.int32)
    for s, k in st.rank_ranges(off, L, own, rank):
        perm[s:s + k] = torch.from_numpy(truth[s:s + k])
    st.gather_perm(perm, off, L, own, world, rank)
    q.put((rank, bool(np.array_equal(perm.numpy(), truth))))
    dist.destroy_process_group()


def test_gloo_subtree_gather_rebuilds_permutation():
    import multiprocessing as mpx
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mpx.get_context("spawn")
    q = ctx.Queue()
    world = 3
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}
