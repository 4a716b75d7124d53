"""Python mirror of the reference meshperm interface, backed by the CUDA library.

Names, argument meaning and error behaviour follow the reference free
functions in /root/reference/proj/core/include/meshperm/*.hpp (cited per
function); contract violations raise ValueError where the reference throws
std::invalid_argument.  Host inputs are numpy int32 arrays; torch CUDA
tensors are accepted wherever a device-resident call makes sense (order()).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import ALLGATHER_FN, LOCAL_MODES, SCHEDULES, MpComm, MpConfig, MpCsr, MpResult, check, lib


# ----------------------------------------------------------------- data model
@dataclass
class TriangleMesh:  # types.hpp:15-18
    vertex_count: int
    triangles: np.ndarray  # (T, 3) int32


@dataclass
class AdjacencyGraph:  # graph.hpp:12-24
    n: int
    offsets: np.ndarray    # int32, n + 1
    neighbors: np.ndarray  # int32, offsets[n]

    def neighbors_of(self, v: int) -> np.ndarray:
        return self.neighbors[self.offsets[v]:self.offsets[v + 1]]

    def edge_count(self) -> int:
        return int(self.offsets[self.n]) // 2


@dataclass
class PatchPartition:  # patching.hpp:11-17
    assignment: np.ndarray
    patch_count: int
    target_size: int = 256


@dataclass
class QuotientGraph:  # quotient.hpp:17-37 (positive edges only)
    patch_count: int
    node_weight: np.ndarray
    edges: list  # sorted (p, q, w), p < q, w > 0

    def positive_edges(self):
        return list(self.edges)


@dataclass
class EliminationTree:  # etree.hpp:19-33, flattened
    n: int
    nd_level: int
    node_offsets: np.ndarray   # 2^(L+1)
    vertices: np.ndarray       # n
    local_perm: np.ndarray | None = None

    def node_count(self) -> int:
        return len(self.node_offsets) - 1

    def node(self, i: int) -> np.ndarray:
        return self.vertices[self.node_offsets[i]:self.node_offsets[i + 1]]

    def node_perm(self, i: int) -> np.ndarray:
        return self.local_perm[self.node_offsets[i]:self.node_offsets[i + 1]]


@dataclass
class Permutation:  # assemble.hpp:12-20
    perm: np.ndarray
    inverse: np.ndarray


@dataclass
class FillReport:  # symbolic.hpp:13-19
    nnz_A: int
    nnz_L: int
    fill_ratio: float
    column_counts: np.ndarray
    cost: int
    parents: np.ndarray | None = None


@dataclass
class PipelineResult:  # pipeline.hpp:56-61
    patch: PatchPartition
    tree: EliminationTree
    perm: Permutation
    fill: FillReport | None
    stage_ms: dict = field(default_factory=dict)
    kernel_launches: int = 0
    kernel_ms: dict = field(default_factory=dict)  # per kernel family (mp_result.kernel_ms)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


# ----------------------------------------------------------------- context
class Context:
    """Owns the device workspace and stream for one GPU (mp_context)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().mp_context_create(C.byref(h), device))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            lib().mp_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        check(lib().mp_context_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))

    TUNING = {"fps_cluster": 0, "fps_qcap": 1, "fps_grid_radius": 2, "fps_grid_cands": 3,
              "fps_sub_region": 4, "lloyd_blocks": 5,
              "lloyd_cluster_n": 6, "md_threads": 7}

    def set_tuning(self, key: str, value: int):
        """mp_context_set_tuning: force a fallback path or a sizing (results unchanged)."""
        check(lib().mp_context_set_tuning(self.handle, self.TUNING[key], int(value)))

    def set_fill_algorithm(self, algo: str):
        """'etree' (default: elimination tree + column counts) or 'game' (the
        elimination game of symbolic.cpp:33-45); identical outputs."""
        check(lib().mp_context_set_fill_algorithm(self.handle, {"etree": 0, "game": 1}[algo]))


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _csr(g: AdjacencyGraph) -> MpCsr:
    off, nbr = _i32(g.offsets), _i32(g.neighbors)
    c = MpCsr(int(g.n), _ptr(off), _ptr(nbr) if nbr.size else C.c_void_p(0), 0)
    c._keep = (off, nbr)  # keep buffers alive
    return c


# ----------------------------------------------------------------- generators (host)
def make_grid_mesh(rows: int, cols: int) -> TriangleMesh:  # pipeline.hpp:63-65
    t = lib().mp_grid_mesh_triangles(rows, cols)
    tris = np.zeros((max(t, 0), 3), np.int32)
    check(lib().mp_make_grid_mesh(rows, cols, _ptr(tris)))
    return TriangleMesh(rows * cols, tris)


def make_random_mesh(rows: int, cols: int, seed: int) -> TriangleMesh:  # tests/test_support.hpp:66-86
    t = lib().mp_grid_mesh_triangles(rows, cols)
    tris = np.zeros((max(t, 0), 3), np.int32)
    check(lib().mp_make_random_mesh(rows, cols, C.c_uint64(seed), _ptr(tris)))
    return TriangleMesh(rows * cols, tris)


def make_torus_mesh(rows: int, cols: int) -> TriangleMesh:
    t = lib().mp_torus_mesh_triangles(rows, cols)
    tris = np.zeros((max(t, 0), 3), np.int32)
    check(lib().mp_make_torus_mesh(rows, cols, _ptr(tris)))
    return TriangleMesh(rows * cols, tris)


def make_icosphere_mesh(f: int) -> TriangleMesh:
    tris = np.zeros((lib().mp_icosphere_triangles(f), 3), np.int32)
    check(lib().mp_make_icosphere_mesh(f, _ptr(tris)))
    return TriangleMesh(int(lib().mp_icosphere_vertices(f)), tris)


def mesh_to_graph(mesh: TriangleMesh) -> AdjacencyGraph:  # graph.hpp:56
    tris = _i32(mesh.triangles).reshape(-1, 3)
    n = int(mesh.vertex_count)
    off = np.zeros(n + 1, np.int32)
    nnz = C.c_int64()
    check(lib().mp_mesh_to_graph(n, len(tris), _ptr(tris), _ptr(off), C.c_void_p(0), C.byref(nnz)))
    nbr = np.zeros(nnz.value, np.int32)
    check(lib().mp_mesh_to_graph(n, len(tris), _ptr(tris), _ptr(off), _ptr(nbr), C.byref(nnz)))
    return AdjacencyGraph(n, off, nbr)


def mesh_to_graph_device(mesh: TriangleMesh, ctx: Context | None = None) -> AdjacencyGraph:
    """graph.hpp:51 mesh_to_graph computed on the GPU; same
    AdjacencyGraph as the reference (sorted, deduplicated, symmetric lists)."""
    ctx = ctx or default_context()
    tris = _i32(mesh.triangles).reshape(-1, 3)
    n = int(mesh.vertex_count)
    off = np.zeros(n + 1, np.int32)
    nnz = C.c_int64()
    check(lib().mp_mesh_to_graph_device(ctx.handle, n, len(tris), _ptr(tris), 0, _ptr(off), C.c_void_p(0), 0,
                                        C.byref(nnz)))
    nbr = np.zeros(nnz.value, np.int32)
    check(lib().mp_mesh_to_graph_device(ctx.handle, n, len(tris), _ptr(tris), 0, _ptr(off), _ptr(nbr), 0,
                                        C.byref(nnz)))
    return AdjacencyGraph(n, off, nbr)


def pattern_to_graph_device(n: int, rows, cols, block_size: int = 1, ctx: Context | None = None) -> AdjacencyGraph:
    """graph.hpp:48 build_graph (block_size 1) / graph.hpp:59 compress_blocks on
    the GPU: a SparsePattern's entries -> the ordering graph."""
    ctx = ctx or default_context()
    rows, cols = _i32(rows), _i32(cols)
    if len(rows) != len(cols):
        raise ValueError("rows and cols differ in length")
    nodes = n // block_size if block_size > 0 and n >= 0 and n % block_size == 0 else 0
    off = np.zeros(nodes + 1, np.int32)
    nnz = C.c_int64()
    f = lib().mp_pattern_to_graph_device
    check(f(ctx.handle, n, len(rows), _ptr(rows), _ptr(cols), 0, block_size, _ptr(off), C.c_void_p(0), 0, C.byref(nnz)))
    nbr = np.zeros(nnz.value, np.int32)
    check(f(ctx.handle, n, len(rows), _ptr(rows), _ptr(cols), 0, block_size, _ptr(off), _ptr(nbr), 0, C.byref(nnz)))
    return AdjacencyGraph(nodes, off, nbr)


def lift_patches(partition: PatchPartition, block_size: int, ctx: Context | None = None) -> PatchPartition:
    """graph.hpp:62 lift_patches: every block row inherits its node's patch."""
    ctx = ctx or default_context()
    a = _i32(partition.assignment)
    out = np.zeros(max(len(a) * block_size, 1), np.int32)
    check(lib().mp_lift_patches(ctx.handle, len(a), _ptr(a), block_size, _ptr(out), 0))
    return PatchPartition(out[:len(a) * block_size], partition.patch_count)


# run_baselines (pipeline.cpp:162-186): the comparison orderings as configs of
# the same path.
BASELINES = {
    "natural": dict(nd_level=0, local_mode="natural"),
    "md": dict(nd_level=0, local_mode="approx_md"),
    "nd-vertex": dict(patch_size=1),
}


def run_baseline(g: AdjacencyGraph, name: str, ctx: Context | None = None, **kw) -> PipelineResult:
    """One run_baselines row: `natural` (identity order), `md` (approximate
    minimum degree on the whole graph) or `nd-vertex` (patch size 1)."""
    if name not in BASELINES:
        raise ValueError("unknown baseline: " + name)
    cfg = dict(kw)
    cfg.update(BASELINES[name])
    return order(g, ctx=ctx, **cfg)


def mesh_to_graph_device_ptr(ctx: Context, nv: int, ntri: int, tris_ptr: int, off_ptr: int, nbr_ptr: int) -> int:
    """Device-pointer form (tris, off, nbr all device memory; nbr capacity
    >= 6 * ntri or the nnz of an earlier call).  Returns nnz."""
    nnz = C.c_int64()
    check(lib().mp_mesh_to_graph_device(ctx.handle, nv, ntri, C.c_void_p(tris_ptr), 1, C.c_void_p(off_ptr),
                                        C.c_void_p(nbr_ptr), 1, C.byref(nnz)))
    return int(nnz.value)


def default_nd_level(n: int) -> int:  # etree.hpp:35-36
    return int(lib().mp_default_nd_level(n))


# ----------------------------------------------------------------- stages
def compute_patches(g: AdjacencyGraph, target_size: int = 256, seed: int = 0,
                    ctx: Context | None = None) -> PatchPartition:  # patching.hpp:26-27
    ctx = ctx or default_context()
    out = np.zeros(max(g.n, 1), np.int32)
    pc = C.c_int32()
    check(lib().mp_compute_patches(ctx.handle, C.byref(_csr(g)), target_size, C.c_uint64(seed), _ptr(out), 0,
                                   C.byref(pc)))
    return PatchPartition(out[:g.n], pc.value, target_size)


def enforce_connectivity(partition: PatchPartition, g: AdjacencyGraph,
                         ctx: Context | None = None) -> PatchPartition:  # patching.hpp:31-32
    ctx = ctx or default_context()
    asg = _i32(partition.assignment)
    if len(asg) != g.n:
        raise ValueError("assignment does not cover the graph")
    out = np.zeros(max(g.n, 1), np.int32)
    pc = C.c_int32()
    check(lib().mp_enforce_connectivity(ctx.handle, C.byref(_csr(g)), _ptr(asg), partition.patch_count, _ptr(out),
                                        0, C.byref(pc)))
    return PatchPartition(out[:g.n], pc.value, partition.target_size)


@dataclass
class PatchReport:  # patching.hpp:35-42
    patch_sizes: np.ndarray
    disconnected_patches: list
    unused_patches: list

    def all_connected(self) -> bool:
        return not self.disconnected_patches

    def clean(self) -> bool:
        return not self.disconnected_patches and not self.unused_patches


def validate_user_patches(partition: PatchPartition, g: AdjacencyGraph,
                          ctx: Context | None = None) -> PatchReport:  # patching.hpp:44-45
    """Diagnostics of a user assignment, computed on the GPU; ValueError with
    the reference's messages for a wrong length or an out-of-range id."""
    ctx = ctx or default_context()
    a = _i32(partition.assignment)
    if len(a) != g.n:
        raise ValueError(f"assignment covers {len(a)} vertices, graph has {g.n}")
    P = int(partition.patch_count)
    sizes = np.zeros(max(P, 1), np.int64)
    dis, unu = np.zeros(max(P, 1), np.int32), np.zeros(max(P, 1), np.int32)
    nd, nu = C.c_int32(), C.c_int32()
    check(lib().mp_validate_user_patches(ctx.handle, C.byref(_csr(g)), _ptr(a), P, _ptr(sizes), _ptr(dis),
                                         C.byref(nd), _ptr(unu), C.byref(nu)))
    return PatchReport(sizes[:P], dis[:nd.value].tolist(), unu[:nu.value].tolist())


def build_quotient(g: AdjacencyGraph, assignment, patch_count: int,
                   ctx: Context | None = None) -> QuotientGraph:  # quotient.hpp:41
    ctx = ctx or default_context()
    asg = _i32(assignment)
    if len(asg) != g.n:
        raise ValueError(f"patch assignment covers {len(asg)} vertices, graph has {g.n}")
    nw = np.zeros(max(patch_count, 1), np.int64)
    ne = C.c_int64()
    csr = _csr(g)
    check(lib().mp_build_quotient(ctx.handle, C.byref(csr), _ptr(asg), patch_count, _ptr(nw), C.c_void_p(0),
                                  C.c_void_p(0), C.c_void_p(0), C.byref(ne)))
    ep = np.zeros(max(ne.value, 1), np.int32)
    eq = np.zeros(max(ne.value, 1), np.int32)
    ew = np.zeros(max(ne.value, 1), np.int64)
    check(lib().mp_build_quotient(ctx.handle, C.byref(csr), _ptr(asg), patch_count, _ptr(nw), _ptr(ep), _ptr(eq),
                                  _ptr(ew), C.byref(ne)))
    m = ne.value
    return QuotientGraph(patch_count, nw[:patch_count],
                         list(zip(ep[:m].tolist(), eq[:m].tolist(), ew[:m].tolist())))


def build_etree(g: AdjacencyGraph, assignment, patch_count: int, nd_level: int, seed: int = 0,
                ctx: Context | None = None) -> EliminationTree:  # etree.hpp:52-53
    ctx = ctx or default_context()
    asg = _i32(assignment)
    if len(asg) != g.n:
        raise ValueError("patch map does not cover the graph")
    if nd_level < 0 or nd_level > 24:
        raise ValueError("nd_level out of range")
    nn = (1 << (nd_level + 1)) - 1
    off = np.zeros(nn + 1, np.int32)
    verts = np.zeros(max(g.n, 1), np.int32)
    check(lib().mp_build_etree(ctx.handle, C.byref(_csr(g)), _ptr(asg), patch_count, nd_level, C.c_uint64(seed),
                               _ptr(off), _ptr(verts), 0))
    return EliminationTree(g.n, nd_level, off, verts[:g.n])


def order_tree_nodes(tree: EliminationTree, g: AdjacencyGraph, mode: str = "approx_md",
                     ctx: Context | None = None) -> EliminationTree:  # local_order.hpp:36
    ctx = ctx or default_context()
    lp = np.zeros(max(g.n, 1), np.int32)
    off, verts = _i32(tree.node_offsets), _i32(tree.vertices)
    check(lib().mp_order_tree_nodes(ctx.handle, C.byref(_csr(g)), tree.nd_level, _ptr(off), _ptr(verts),
                                    LOCAL_MODES[mode], _ptr(lp), 0))
    tree.local_perm = lp[:g.n]
    return tree


def order_subtrees(tree: EliminationTree, g: AdjacencyGraph, node_mask, local_perm, perm,
                   mode: str = "approx_md", schedule: str = "postorder", ctx: Context | None = None):
    """mp_order_subtrees on host arrays: local_perm / perm entries of the masked
    nodes are written in place (int32 arrays of length n), others untouched."""
    ctx = ctx or default_context()
    nn = (1 << (tree.nd_level + 1)) - 1
    mask = np.ascontiguousarray(node_mask, np.uint8)
    if mask.shape != (nn,):
        raise ValueError("node_mask needs one entry per tree node")
    for a in (local_perm, perm):
        if a.dtype != np.int32 or a.shape != (g.n,) or not a.flags.c_contiguous:
            raise ValueError("local_perm / perm must be contiguous int32 arrays of length n")
    off, verts = _i32(tree.node_offsets), _i32(tree.vertices)
    check(lib().mp_order_subtrees(ctx.handle, C.byref(_csr(g)), tree.nd_level, _ptr(off), _ptr(verts),
                                  LOCAL_MODES[mode], SCHEDULES[schedule], _ptr(mask), _ptr(local_perm), _ptr(perm), 0))


def _schedule_nodes(tree: EliminationTree, schedule) -> np.ndarray:
    """A named schedule (schedule_postorder / schedule_levelorder,
    assemble.hpp:25-29) or any node sequence, as int32 node ids."""
    if isinstance(schedule, str):
        if schedule not in SCHEDULES:
            raise ValueError("unknown schedule: " + schedule)
        return _i32(schedule_nodes(tree.nd_level, schedule))
    return _i32(schedule)


def _nonempty(a: np.ndarray) -> np.ndarray:
    return a if a.size else np.zeros(1, np.int32)


def schedule_nodes(nd_level: int, kind: str = "postorder") -> list[int]:
    """schedule_postorder (left, right, node) / schedule_levelorder (deepest
    level first), assemble.cpp:24-46."""
    nn = (1 << (nd_level + 1)) - 1
    if kind == "levelorder":
        return [i for lev in range(nd_level, -1, -1) for i in range((1 << lev) - 1, (1 << (lev + 1)) - 1)]
    out, st = [], [(0, 0)]
    while st:
        i, state = st.pop()
        if i >= nn:
            continue
        if state == 0:
            st += [(i, 1), (2 * i + 1, 0)]
        elif state == 1:
            st += [(i, 2), (2 * i + 2, 0)]
        else:
            out.append(i)
    return out


def validate_schedule(tree: EliminationTree, sequence) -> int | None:
    """assemble.hpp:35 validate_schedule: the first violating position, or None."""
    seq = _i32(sequence)
    bad = C.c_int64()
    check(lib().mp_validate_schedule(tree.nd_level, C.c_void_p(_nonempty(seq).ctypes.data), len(seq), C.byref(bad)))
    return None if bad.value < 0 else int(bad.value)


def compute_perm(tree: EliminationTree, g: AdjacencyGraph, schedule="postorder",
                 ctx: Context | None = None) -> Permutation:  # assemble.hpp:25-38
    """compute_perm(tree, g, schedule): `schedule` is "postorder",
    "levelorder" or any node sequence (validated like validate_schedule;
    ValueError "invalid schedule at position N")."""
    ctx = ctx or default_context()
    if tree.n != g.n:
        raise ValueError("tree was built for a different graph")
    if tree.local_perm is None:
        raise ValueError("tree nodes have no local order")
    pm = np.zeros(max(g.n, 1), np.int32)
    inv = np.zeros(max(g.n, 1), np.int32)
    sched = _schedule_nodes(tree, schedule)
    check(lib().mp_compute_perm_schedule(ctx.handle, g.n, tree.nd_level, _ptr(_i32(tree.node_offsets)),
                                         _ptr(_i32(tree.vertices)), _ptr(_i32(tree.local_perm)),
                                         C.c_void_p(_nonempty(sched).ctypes.data), len(sched), _ptr(pm), _ptr(inv), 0))
    return Permutation(pm[:g.n], inv[:g.n])


def tree_separation_violations(g: AdjacencyGraph, tree: EliminationTree, ctx: Context | None = None) -> int:
    """edges joining tree nodes that are neither equal nor
    ancestor-related (tests/etree_test.cpp:171-179).  0 implies the
    reference's pipeline self-check cross_block_fill == 0 (pipeline.cpp:141)."""
    ctx = ctx or default_context()
    v = C.c_int64()
    check(lib().mp_tree_separation_check(ctx.handle, C.byref(_csr(g)), tree.nd_level, _ptr(_i32(tree.node_offsets)),
                                         _ptr(_i32(tree.vertices)), 0, C.byref(v)))
    return int(v.value)


def tree_fill(g: AdjacencyGraph, tree: EliminationTree, schedule="postorder",
              ctx: Context | None = None) -> FillReport:  # symbolic.hpp:23 + :31
    """elimination_fill + factor_etree_parents of compute_perm(tree, g,
    schedule), played subtree by subtree on the device (any valid schedule)."""
    ctx = ctx or default_context()
    cc = np.zeros(max(g.n, 1), np.int64)
    par = np.zeros(max(g.n, 1), np.int32)
    a, l, c = C.c_int64(), C.c_int64(), C.c_int64()
    r = C.c_double()
    sched = _schedule_nodes(tree, schedule)
    check(lib().mp_tree_fill_schedule(ctx.handle, C.byref(_csr(g)), tree.nd_level, _ptr(_i32(tree.node_offsets)),
                                      _ptr(_i32(tree.vertices)), _ptr(_i32(tree.local_perm)),
                                      C.c_void_p(_nonempty(sched).ctypes.data), len(sched), _ptr(cc), _ptr(par), 0,
                                      C.byref(a),
                                      C.byref(l), C.byref(c), C.byref(r)))
    return FillReport(a.value, l.value, r.value, cc[:g.n], c.value, par[:g.n])


def _perm_array(g: AdjacencyGraph, perm) -> np.ndarray:
    p = _i32(perm.perm if isinstance(perm, Permutation) else perm)
    if len(p) != g.n:  # symbolic.cpp:12-14
        raise ValueError("permutation does not match the graph")
    return p


def elimination_fill(g: AdjacencyGraph, perm, ctx: Context | None = None) -> FillReport:  # symbolic.hpp:23
    """The elimination game for ANY permutation (new position -> old index),
    on the device; FillReport.parents = factor_etree_parents (symbolic.hpp:31)."""
    ctx = ctx or default_context()
    p = _perm_array(g, perm)
    cc = np.zeros(max(g.n, 1), np.int64)
    par = np.zeros(max(g.n, 1), np.int32)
    a, l, c = C.c_int64(), C.c_int64(), C.c_int64()
    r = C.c_double()
    check(lib().mp_elimination_fill(ctx.handle, C.byref(_csr(g)), _ptr(p), _ptr(cc), _ptr(par), 0, C.byref(a),
                                    C.byref(l), C.byref(c), C.byref(r)))
    return FillReport(a.value, l.value, r.value, cc[:g.n], c.value, par[:g.n])


def factor_etree_parents(g: AdjacencyGraph, perm, ctx: Context | None = None) -> np.ndarray:  # symbolic.hpp:31
    return elimination_fill(g, perm, ctx).parents


def cross_block_fill(g: AdjacencyGraph, perm, tree: EliminationTree, ctx: Context | None = None) -> int:
    """symbolic.hpp:37: factor entries joining unrelated tree nodes (exact count)."""
    ctx = ctx or default_context()
    p = _perm_array(g, perm)
    if tree.n != g.n:
        raise ValueError("tree was built for a different graph")
    v = C.c_int64()
    check(lib().mp_cross_block_fill(ctx.handle, C.byref(_csr(g)), _ptr(p), tree.nd_level,
                                    _ptr(_i32(tree.node_offsets)), _ptr(_i32(tree.vertices)), 0, C.byref(v)))
    return int(v.value)


# ----------------------------------------------------------------- whole path
def make_config(patch_size=256, nd_level=-1, seed=0, local_mode="approx_md", schedule="postorder", block_size=1,
                want_fill=True) -> MpConfig:
    return MpConfig(patch_size, nd_level, seed, LOCAL_MODES[local_mode], SCHEDULES[schedule], block_size,
                    1 if want_fill else 0)


def _prepare(g: AdjacencyGraph, nd_level: int, block_size: int, want_fill: bool):
    L = nd_level if nd_level >= 0 else default_nd_level(g.n)
    nn = (1 << (L + 1)) - 1
    N = block_size * g.n
    bufs = {
        "patch_of": np.zeros(max(g.n, 1), np.int32),
        "tree_node_offsets": np.zeros(nn + 1, np.int32),
        "tree_vertices": np.zeros(max(N, 1), np.int32),
        "tree_local_perm": np.zeros(max(N, 1), np.int32),
        "perm": np.zeros(max(N, 1), np.int32),
        "inverse": np.zeros(max(N, 1), np.int32),
        "etree_parent": np.zeros(max(N, 1), np.int32),
        "column_counts": np.zeros(max(N, 1), np.int64),
    }
    res = MpResult()
    res.on_device = 0
    for k, v in bufs.items():
        setattr(res, k, _ptr(v))
    if not want_fill:
        res.etree_parent = None
        res.column_counts = None
    return bufs, res


KERNEL_NAMES = ["fps", "lloyd", "fm", "refine", "md", "symbolic"]


def _finish(g: AdjacencyGraph, bufs, res: MpResult, patch_size: int, block_size: int, want_fill: bool):
    N = block_size * g.n
    tree = EliminationTree(N, res.nd_level, bufs["tree_node_offsets"], bufs["tree_vertices"][:N],
                           bufs["tree_local_perm"][:N])
    fill = None
    if want_fill:
        fill = FillReport(res.nnz_A, res.nnz_L, res.fill_ratio, bufs["column_counts"][:N], res.cost,
                          bufs["etree_parent"][:N])
    names = ["patch", "quotient", "etree", "local", "assemble", "symbolic"]
    return PipelineResult(PatchPartition(bufs["patch_of"][:g.n], res.patch_count, patch_size), tree,
                          Permutation(bufs["perm"][:N], bufs["inverse"][:N]), fill,
                          {k: float(res.stage_ms[i]) for i, k in enumerate(names)}, int(res.kernel_launches),
                          {k: float(res.kernel_ms[i]) for i, k in enumerate(KERNEL_NAMES)})


def order(g: AdjacencyGraph, patch_size: int = 256, nd_level: int = -1, seed: int = 0, local_mode="approx_md",
          schedule="postorder", block_size: int = 1, want_fill: bool = True,
          ctx: Context | None = None, user_patches: PatchPartition | None = None) -> PipelineResult:
    """run_pipeline's ordering stages (pipeline.cpp:100-140) on host arrays.
    `user_patches` is the RunConfig.patch_file path (pipeline.cpp:102-111): the
    given GroupMap is validated and its disconnected patches split instead of
    computing patches."""
    ctx = ctx or default_context()
    custom = None if isinstance(schedule, str) else _i32(schedule)
    cfg = make_config(patch_size, nd_level, seed, local_mode, "postorder" if custom is not None else schedule,
                      block_size, want_fill)
    if custom is not None:  # compute_perm(tree, g, schedule) with a caller sequence (assemble.hpp:37)
        buf = custom if custom.size else np.zeros(1, np.int32)  # non-NULL even when empty
        cfg.schedule_nodes = C.c_void_p(buf.ctypes.data)
        cfg.schedule_len = len(custom)
    if user_patches is not None:
        up = _i32(user_patches.assignment)
        if len(up) != g.n:  # patching.cpp:387-390
            raise ValueError(f"assignment covers {len(up)} vertices, graph has {g.n}")
        cfg.user_patches = _ptr(up)
        cfg.user_patch_count = int(user_patches.patch_count)
    bufs, res = _prepare(g, nd_level, block_size, want_fill)
    check(lib().mp_order(ctx.handle, C.byref(_csr(g)), C.byref(cfg), C.byref(res)))
    r = _finish(g, bufs, res, patch_size, block_size, want_fill)
    r.work = [int(res.work[i]) for i in range(16)]
    return r


def order_batch(graphs, contexts, patch_size: int = 256, nd_level: int = -1, seed: int = 0,
                local_mode="approx_md", schedule="postorder", block_size: int = 1,
                want_fill: bool = True) -> list[PipelineResult]:
    """mp_order_batch: every graph ordered (same config), frames spread over
    `contexts` (host threads + streams inside the library); results equal
    sequential order() calls, in input order."""
    graphs = list(graphs)
    cfg = make_config(patch_size, nd_level, seed, local_mode, schedule, block_size, want_fill)
    preps = [_prepare(g, nd_level, block_size, want_fill) for g in graphs]
    keep = [_csr(g) for g in graphs]  # the struct copies below do not own the arrays
    csrs = (MpCsr * max(len(graphs), 1))(*keep)
    cfgs = (MpConfig * max(len(graphs), 1))(*[cfg for _ in graphs])
    ress = (MpResult * max(len(graphs), 1))(*[r for _, r in preps])
    handles = (C.c_void_p * len(contexts))(*[c.handle for c in contexts])
    status = np.zeros(max(len(graphs), 1), np.int32)
    check(lib().mp_order_batch(handles, len(contexts), len(graphs), csrs, cfgs, ress, _ptr(status)))
    return [_finish(g, bufs, ress[i], patch_size, block_size, want_fill)
            for i, (g, (bufs, _)) in enumerate(zip(graphs, preps))]


def order_device(ctx: Context, n: int, offsets_ptr: int, neighbors_ptr: int, out: dict, patch_size=256,
                 nd_level=-1, seed=0, local_mode="approx_md", schedule="postorder", block_size=1,
                 want_fill=True) -> MpResult:
    """mp_order on device-resident CSR and device output pointers (dict of name -> ptr)."""
    cfg = make_config(patch_size, nd_level, seed, local_mode, schedule, block_size, want_fill)
    csr = MpCsr(n, C.c_void_p(offsets_ptr), C.c_void_p(neighbors_ptr), 1)
    res = MpResult()
    res.on_device = 1
    for k, v in out.items():
        setattr(res, k, C.c_void_p(v))
    check(lib().mp_order(ctx.handle, C.byref(csr), C.byref(cfg), C.byref(res)))
    return res


# ----------------------------------------------------------------- multi-GPU (C3)
class Comm:
    """mp_comm: this rank, the world size and an all-gather.

    * Comm.nccl(rank, world, device, unique_id): the library's own NCCL
      communicator (device buffers on the context's stream); rank 0 makes
      the id with Comm.nccl_unique_id() and ships it to the others.
    * Comm.from_allgather(rank, world, fn): fn(send: bytes) -> bytes of
      world * len(send), rank-major (host buffers: gloo, MPI, threads ...).
    * Comm.torch_distributed(): from_allgather over the current
      torch.distributed group (CPU tensors, e.g. the gloo backend).
    """

    def __init__(self):
        self.struct = MpComm()
        self._fn = None
        self._nccl = False

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        check(lib().mp_nccl_get_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, rank: int, world: int, device: int, unique_id: bytes) -> "Comm":
        c = cls()
        uid = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        check(lib().mp_nccl_comm_init(C.byref(c.struct), uid, world, rank, device))
        c._nccl = True
        return c

    @classmethod
    def from_allgather(cls, rank: int, world: int, fn) -> "Comm":
        c = cls()

        def trampoline(user, send, recv, nbytes, stream):
            try:
                data = C.string_at(send, nbytes) if nbytes else b""
                got = fn(data)
                if len(got) != world * nbytes:
                    return 1
                if got:
                    C.memmove(recv, got, len(got))
                return 0
            except Exception:  # never raise across the C boundary
                return 2

        c._fn = ALLGATHER_FN(trampoline)
        c.struct.rank, c.struct.world, c.struct.device_buffers = rank, world, 0
        c.struct.allgather = C.cast(c._fn, C.c_void_p)
        c.struct.user = None
        return c

    @classmethod
    def torch_distributed(cls, group=None) -> "Comm":
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def fn(data: bytes) -> bytes:
            t = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.empty(0, dtype=torch.uint8)
            out = torch.empty(world * len(data), dtype=torch.uint8)
            dist.all_gather_into_tensor(out, t, group=group)
            return out.numpy().tobytes()

        return cls.from_allgather(rank, world, fn)

    def close(self):
        if self._nccl:
            lib().mp_nccl_comm_destroy(C.byref(self.struct))
            self._nccl = False


def order_sharded(g: AdjacencyGraph, comm: Comm, patch_size: int = 256, nd_level: int = -1, seed: int = 0,
                  local_mode="approx_md", schedule="postorder", want_fill: bool = True,
                  ctx: Context | None = None) -> PipelineResult:
    """mp_order_sharded: one mesh ordered by `comm.world` ranks together (each
    calls this with the same graph); every rank returns the complete result,
    identical to order()."""
    ctx = ctx or default_context()
    cfg = make_config(patch_size, nd_level, seed, local_mode, schedule if isinstance(schedule, str) else "postorder",
                      1, want_fill)
    custom = None if isinstance(schedule, str) else _nonempty(_i32(schedule))
    if custom is not None:
        cfg.schedule_nodes = C.c_void_p(custom.ctypes.data)
        cfg.schedule_len = len(schedule)
    bufs, res = _prepare(g, nd_level, 1, want_fill)
    check(lib().mp_order_sharded(ctx.handle, C.byref(_csr(g)), C.byref(cfg), C.byref(comm.struct), C.byref(res)))
    r = _finish(g, bufs, res, patch_size, 1, want_fill)
    r.work = [int(res.work[i]) for i in range(16)]
    return r
