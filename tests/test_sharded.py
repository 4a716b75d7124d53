"""mp_order_sharded (SURVEY §8e, configs[2]): one mesh ordered by several
ranks, each on its own context, exchanging node sizes, the owned nodes' tree
lists, the subtree roots' live elements and the owned column counts through
mp_comm's all-gather.  Every rank must return exactly mp_order's result.

All ranks share the one GPU of the test box; the collective is the caller's
host all-gather (threads in one process, or gloo across processes), the
library's NCCL one at world 1.  The CPU tests check the host all-gather
plumbing (Comm.from_allgather / Comm.torch_distributed) under gloo.
"""
import ctypes as C
import socket
import threading

import numpy as np
import pytest

import paper_2602_00898_b200 as mp
from paper_2602_00898_b200._lib import ALLGATHER_FN


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class ThreadAllGather:
    """An in-process all-gather for `world` threads (host buffers)."""

    def __init__(self, world):
        self.world, self.parts = world, [None] * world
        self.b1, self.b2 = threading.Barrier(world), threading.Barrier(world)

    def comm(self, rank):
        def fn(data):
            self.parts[rank] = data
            self.b1.wait()
            out = b"".join(self.parts)
            self.b2.wait()
            return out
        return mp.Comm.from_allgather(rank, self.world, fn)


def _same(a, b, fill=True):
    assert a.patch.patch_count == b.patch.patch_count
    assert np.array_equal(a.patch.assignment, b.patch.assignment)
    assert np.array_equal(a.tree.node_offsets, b.tree.node_offsets)
    assert np.array_equal(a.tree.vertices, b.tree.vertices)
    assert np.array_equal(a.tree.local_perm, b.tree.local_perm)
    assert np.array_equal(a.perm.perm, b.perm.perm) and np.array_equal(a.perm.inverse, b.perm.inverse)
    if fill:
        assert (a.fill.nnz_L, a.fill.cost, a.fill.nnz_A) == (b.fill.nnz_L, b.fill.cost, b.fill.nnz_A)
        assert np.array_equal(a.fill.column_counts, b.fill.column_counts)
        assert np.array_equal(a.fill.parents, b.fill.parents)


def _run_threads(g, world, **kw):
    ag = ThreadAllGather(world)
    ctxs = [mp.Context(0) for _ in range(world)]
    out, err = [None] * world, []

    def work(r):
        try:
            out[r] = mp.order_sharded(g, ag.comm(r), ctx=ctxs[r], **kw)
        except Exception as e:  # pragma: no cover - reported below
            err.append((r, e))
            ag.b1.abort(), ag.b2.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for c in ctxs:
        c.close()
    assert not err, err
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sharded_threads_equal_single_gpu(world):
    g = mp.mesh_to_graph(mp.make_icosphere_mesh(40))  # n = 16,002, L = 4
    ref = mp.order(g)
    outs = _run_threads(g, world)
    owned = 0
    for r in outs:
        _same(r, ref)
        owned += r.work[15]
    top = int(ref.tree.node_offsets[(1 << min(ref.tree.nd_level, int(np.ceil(np.log2(world))))) - 1])
    assert owned == g.n + (world - 1) * top  # subtrees split between ranks, top replicated


@pytest.mark.gpu
@pytest.mark.parametrize("world,kw", [(2, dict(schedule="levelorder")), (4, dict(local_mode="exact_md")),
                                      (3, dict(patch_size=64, nd_level=6)), (2, dict(want_fill=False))])
def test_sharded_configs_match(world, kw):
    g = mp.mesh_to_graph(mp.make_random_mesh(150, 140, 9))
    ref = mp.order(g, **kw)
    for r in _run_threads(g, world, **kw):
        _same(r, ref, fill=kw.get("want_fill", True))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_small_and_disconnected_graphs(world):
    """Trees that stop above the shard level, several components."""
    a = mp.mesh_to_graph(mp.make_grid_mesh(40, 40))
    b = mp.mesh_to_graph(mp.make_grid_mesh(9, 7))
    off = np.concatenate([a.offsets, a.offsets[-1] + b.offsets[1:]]).astype(np.int32)
    nbr = np.concatenate([a.neighbors, b.neighbors + a.n]).astype(np.int32)
    for g, kw in ((mp.AdjacencyGraph(a.n + b.n, off, nbr), dict(patch_size=40, nd_level=3)),
                  (mp.mesh_to_graph(mp.make_grid_mesh(8, 8)), dict()),
                  (mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), dict(patch_size=900, nd_level=3))):
        ref = mp.order(g, **kw)
        for r in _run_threads(g, world, **kw):
            _same(r, ref)


@pytest.mark.gpu
def test_sharded_nccl_world_1():
    g = mp.mesh_to_graph(mp.make_grid_mesh(90, 70))
    comm = mp.Comm.nccl(0, 1, 0, mp.Comm.nccl_unique_id())
    try:
        r = mp.order_sharded(g, comm)
    finally:
        comm.close()
    _same(r, mp.order(g))


def _gloo_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    import paper_2602_00898_b200 as mp
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = mp.mesh_to_graph(mp.make_icosphere_mesh(30))
    r = mp.order_sharded(g, mp.Comm.torch_distributed())
    import hashlib
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    q.put((rank, dg(r.perm.perm), dg(r.fill.column_counts), dg(r.fill.parents), int(r.fill.nnz_L)))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_gloo_processes_world_2():
    import hashlib
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port, world = _port(), 2
    ps = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict((x[0], x[1:]) for x in (q.get(timeout=300) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = mp.mesh_to_graph(mp.make_icosphere_mesh(30))
    ref = mp.order(g)
    dg = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    want = (dg(ref.perm.perm), dg(ref.fill.column_counts), dg(ref.fill.parents), int(ref.fill.nnz_L))
    assert got == {0: want, 1: want}


# ---------------------------------------------------------------- CPU: host all-gather plumbing
def _plumbing_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    import paper_2602_00898_b200 as mp
    from paper_2602_00898_b200._lib import ALLGATHER_FN
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = mp.Comm.torch_distributed()
    fn = C.cast(comm.struct.allgather, ALLGATHER_FN)
    res = []
    for n in (0, 5, 64):  # the library calls it with host buffers exactly like this
        send = np.arange(n, dtype=np.int32) + 1000 * rank
        recv = np.full(n * world, -1, np.int32)
        rc = fn(None, send.ctypes.data if n else None, recv.ctypes.data if n else None, 4 * n, None)
        res.append((rc, recv.tolist()))
    q.put((rank, comm.struct.rank, comm.struct.world, res))
    dist.destroy_process_group()


def test_host_allgather_comm_under_gloo():
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port, world = _port(), 2
    ps = [ctx.Process(target=_plumbing_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict((x[0], x[1:]) for x in (q.get(timeout=120) for _ in ps))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        rk, ws, res = got[r]
        assert (rk, ws) == (r, world)
        for n, (rc, recv) in zip((0, 5, 64), res):
            assert rc == 0
            assert recv == [v for q_ in range(world) for v in (np.arange(n) + 1000 * q_).tolist()]


def test_thread_allgather_comm():
    world = 3
    ag = ThreadAllGather(world)
    out = [None] * world

    def w(r):
        c = ag.comm(r)
        fn = C.cast(c.struct.allgather, ALLGATHER_FN)
        send = np.array([r, r + 10], np.int64)
        recv = np.zeros(2 * world, np.int64)
        out[r] = (fn(None, send.ctypes.data, recv.ctypes.data, 16, None), recv.tolist())

    ts = [threading.Thread(target=w, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(o == (0, [0, 10, 1, 11, 2, 12]) for o in out)
