"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU oracles.

* ``Restatement``: oracle/_ref/libmp_oracle.so, the plain-C restatement of the
  reference ordering path (oracle/mp_oracle.c).
* ``Reference``: oracle/_ref/libmeshperm_ref.so, the unmodified reference
  meshperm core compiled from /root/reference by oracle/Makefile, behind
  oracle/ref_shim.cpp.

Both expose the same methods, so parity tests can run either.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
RESTATEMENT_SO = REF_DIR / "libmp_oracle.so"
REFERENCE_SO = REF_DIR / "libmeshperm_ref.so"


def build(quiet: bool = True) -> None:
    """Build what can be built here (the reference only where /root/reference exists)."""
    subprocess.run(["make", "-C", str(HERE), "-j8"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class _Base:
    prefix = ""
    path: Path

    def __init__(self):
        if not self.path.exists():
            raise FileNotFoundError(f"{self.path} missing; run `make -C oracle`")
        self.lib = C.CDLL(str(self.path))
        getattr(self.lib, self.prefix + "last_error").restype = C.c_char_p

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, rc):
        if rc != 0:
            msg = self._f("last_error")().decode()
            raise ValueError(msg)

    # --- stages -------------------------------------------------------------
    def default_nd_level(self, n):
        f = self._f("default_nd_level")
        f.restype = C.c_int32
        return f(C.c_int32(n))

    def compute_patches(self, g, target=256, seed=0):
        out = np.zeros(max(g.n, 1), np.int32)
        pc = C.c_int32()
        self._check(self._f("compute_patches")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                               C.c_int32(target), C.c_uint64(seed), _p(out), C.byref(pc)))
        return out[:g.n], pc.value

    def enforce_connectivity(self, g, assignment, patch_count):
        out = np.zeros(max(g.n, 1), np.int32)
        pc = C.c_int32()
        self._check(self._f("enforce_connectivity")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                                    _p(_i32(assignment)), C.c_int32(patch_count), _p(out),
                                                    C.byref(pc)))
        return out[:g.n], pc.value

    def build_quotient(self, g, assignment, patch_count):
        nw = np.zeros(max(patch_count, 1), np.int64)
        ne = C.c_int64()
        args = [C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)), _p(_i32(assignment)),
                C.c_int32(patch_count)]
        self._check(self._f("build_quotient")(*args, _p(nw), None, None, None, C.byref(ne)))
        m = ne.value
        ep, eq, ew = np.zeros(max(m, 1), np.int32), np.zeros(max(m, 1), np.int32), np.zeros(max(m, 1), np.int64)
        self._check(self._f("build_quotient")(*args, _p(nw), _p(ep), _p(eq), _p(ew), C.byref(ne)))
        return nw[:patch_count], list(zip(ep[:m].tolist(), eq[:m].tolist(), ew[:m].tolist()))

    def build_etree(self, g, assignment, patch_count, nd_level, seed=0):
        nn = (1 << (nd_level + 1)) - 1
        off = np.zeros(nn + 1, np.int32)
        verts = np.zeros(max(g.n, 1), np.int32)
        self._check(self._f("build_etree")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                           _p(_i32(assignment)), C.c_int32(patch_count), C.c_int32(nd_level),
                                           C.c_uint64(seed), _p(off), _p(verts)))
        return off, verts[:g.n]

    def order_tree_nodes(self, g, nd_level, node_offsets, node_vertices, mode=0, threads=1):
        lp = np.zeros(max(g.n, 1), np.int32)
        args = [C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)), C.c_int32(nd_level),
                _p(_i32(node_offsets)), _p(_i32(node_vertices)), C.c_int32(mode)]
        if self.prefix == "ref_":
            args.append(C.c_int32(threads))
        self._check(self._f("order_tree_nodes")(*args, _p(lp)))
        return lp[:g.n]

    def minimum_degree(self, g, mode=0):
        out = np.zeros(max(g.n, 1), np.int32)
        self._check(self._f("minimum_degree")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                              C.c_int32(mode), _p(out)))
        return out[:g.n]

    def compute_perm(self, g, nd_level, node_offsets, node_vertices, local_perm, levelorder=0):
        pm = np.zeros(max(g.n, 1), np.int32)
        inv = np.zeros(max(g.n, 1), np.int32)
        if self.prefix == "ref_":
            rc = self._f("compute_perm")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                         C.c_int32(nd_level), _p(_i32(node_offsets)), _p(_i32(node_vertices)),
                                         _p(_i32(local_perm)), C.c_int32(levelorder), _p(pm), _p(inv))
        else:
            rc = self._f("compute_perm")(C.c_int32(g.n), C.c_int32(nd_level), _p(_i32(node_offsets)),
                                         _p(_i32(node_vertices)), _p(_i32(local_perm)), C.c_int32(levelorder),
                                         _p(pm), _p(inv))
        self._check(rc)
        return pm[:g.n], inv[:g.n]

    def elimination_fill(self, g, perm):
        cc = np.zeros(max(g.n, 1), np.int64)
        a, l, c = C.c_int64(), C.c_int64(), C.c_int64()
        if self.prefix == "ref_":
            r = C.c_double()
            rc = self._f("elimination_fill")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                             _p(_i32(perm)), _p(cc), C.byref(a), C.byref(l), C.byref(c), C.byref(r))
        else:
            rc = self._f("elimination_fill")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                             _p(_i32(perm)), _p(cc), C.byref(a), C.byref(l), C.byref(c))
        self._check(rc)
        return dict(nnz_A=a.value, nnz_L=l.value, cost=c.value, column_counts=cc[:g.n])

    def factor_etree_parents(self, g, perm):
        par = np.zeros(max(g.n, 1), np.int32)
        self._check(self._f("factor_etree_parents")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                                    _p(_i32(perm)), _p(par)))
        return par[:g.n]

    # --- the ordering path, stage by stage ------------------------------------
    def order(self, g, patch_size=256, nd_level=-1, seed=0, mode=0, levelorder=0, threads=1):
        """compute_patches -> build_etree -> order_tree_nodes -> compute_perm (pipeline.cpp:100-138)."""
        L = nd_level if nd_level >= 0 else self.default_nd_level(g.n)
        t0 = time.perf_counter()
        asg, pc = self.compute_patches(g, patch_size, seed)
        off, verts = self.build_etree(g, asg, pc, L, seed)
        lp = self.order_tree_nodes(g, L, off, verts, mode, threads)
        pm, inv = self.compute_perm(g, L, off, verts, lp, levelorder)
        ms = (time.perf_counter() - t0) * 1e3
        return dict(assignment=asg, patch_count=pc, nd_level=L, node_offsets=off, node_vertices=verts,
                    local_perm=lp, perm=pm, inverse=inv, ms=ms)


class Restatement(_Base):
    prefix = "mpo_"
    path = RESTATEMENT_SO

    def mesh_to_graph(self, nv, tris):
        tris = _i32(tris).reshape(-1, 3)
        off = np.zeros(nv + 1, np.int32)
        nnz = C.c_int64()
        self._check(self._f("graph_from_triangles")(C.c_int32(nv), C.c_int64(len(tris)), _p(tris), _p(off), None,
                                                    C.byref(nnz)))
        nbr = np.zeros(nnz.value, np.int32)
        self._check(self._f("graph_from_triangles")(C.c_int32(nv), C.c_int64(len(tris)), _p(tris), _p(off),
                                                    _p(nbr), C.byref(nnz)))
        return off, nbr


class Reference(_Base):
    prefix = "ref_"
    path = REFERENCE_SO

    def mesh_to_graph(self, nv, tris):
        tris = _i32(tris).reshape(-1, 3)
        off = np.zeros(nv + 1, np.int32)
        nnz = C.c_int64()
        self._check(self._f("mesh_to_graph")(C.c_int32(nv), C.c_int64(len(tris)), _p(tris), _p(off), None,
                                             C.byref(nnz)))
        nbr = np.zeros(nnz.value, np.int32)
        self._check(self._f("mesh_to_graph")(C.c_int32(nv), C.c_int64(len(tris)), _p(tris), _p(off), _p(nbr),
                                             C.byref(nnz)))
        return off, nbr

    def make_grid_mesh(self, rows, cols):
        """pipeline.cpp:38-55 -> (T, 3) int32 triangles."""
        tris = np.zeros((max(2 * (rows - 1) * (cols - 1), 1), 3), np.int32)
        self._check(self._f("make_grid_mesh")(C.c_int32(rows), C.c_int32(cols), _p(tris)))
        return tris[:2 * (rows - 1) * (cols - 1)]

    def random_mesh(self, rows, cols, seed):
        """tests/test_support.hpp:66-86 mtest::random_mesh -> (T, 3) int32 triangles."""
        tris = np.zeros((max(2 * (rows - 1) * (cols - 1), 1), 3), np.int32)
        self._check(self._f("random_mesh")(C.c_int32(rows), C.c_int32(cols), C.c_uint64(seed), _p(tris)))
        return tris[:2 * (rows - 1) * (cols - 1)]

    def pattern_to_graph(self, n, rows, cols, block_size=1):
        """graph.cpp:53-61 build_graph / :77-94 compress_blocks."""
        rows, cols = _i32(rows), _i32(cols)
        nodes = n // block_size if block_size > 0 else 0
        off = np.zeros(nodes + 1, np.int32)
        nnz = C.c_int64()
        f = self._f("pattern_to_graph")
        self._check(f(C.c_int32(n), C.c_int64(len(rows)), _p(rows), _p(cols), C.c_int32(block_size), _p(off), None,
                      C.byref(nnz)))
        nbr = np.zeros(nnz.value, np.int32)
        self._check(f(C.c_int32(n), C.c_int64(len(rows)), _p(rows), _p(cols), C.c_int32(block_size), _p(off),
                      _p(nbr), C.byref(nnz)))
        return off, nbr

    # --- on-disk formats (io.cpp) -------------------------------------------
    def parse_mesh(self, path, fmt=0):
        """io.cpp:88-184 parse_off (fmt 1) / parse_obj (2) / parse_mesh (0) -> (nv, tris)."""
        nv, nt = C.c_int32(), C.c_int64()
        f = self._f("parse_mesh")
        self._check(f(os.fsencode(path), C.c_int32(fmt), C.byref(nv), C.byref(nt), None))
        tris = np.zeros((nt.value, 3), np.int32)
        self._check(f(os.fsencode(path), C.c_int32(fmt), C.byref(nv), C.byref(nt), _p(tris)))
        return nv.value, tris

    def parse_matrix_market(self, path):
        """io.cpp:186-240 -> (n, rows, cols) of the symmetrized pattern."""
        n, nnz = C.c_int32(), C.c_int64()
        f = self._f("parse_matrix_market")
        self._check(f(os.fsencode(path), C.byref(n), C.byref(nnz), None, None))
        rows, cols = np.zeros(max(nnz.value, 1), np.int32), np.zeros(max(nnz.value, 1), np.int32)
        self._check(f(os.fsencode(path), C.byref(n), C.byref(nnz), _p(rows), _p(cols)))
        return n.value, rows[:nnz.value], cols[:nnz.value]

    def read_patch_file(self, path, n):
        """io.cpp:242-262 -> (assignment, patch_count)."""
        a, pc = np.zeros(max(n, 1), np.int32), C.c_int32()
        self._check(self._f("read_patch_file")(os.fsencode(path), C.c_int32(n), _p(a), C.byref(pc)))
        return a[:n], pc.value

    def write_permutation(self, path, perm):
        """io.cpp:264-268."""
        perm = _i32(perm)
        self._check(self._f("write_permutation")(os.fsencode(path), C.c_int32(len(perm)), _p(perm)))

    def read_permutation(self, path):
        """io.cpp:270-281."""
        n = C.c_int32()
        f = self._f("read_permutation")
        self._check(f(os.fsencode(path), C.byref(n), None))
        p = np.zeros(max(n.value, 1), np.int32)
        self._check(f(os.fsencode(path), C.byref(n), _p(p)))
        return p[:n.value]

    def write_etree(self, path, n, nd_level, node_offsets, node_vertices):
        """io.cpp:283-293."""
        self._check(self._f("write_etree")(os.fsencode(path), C.c_int32(n), C.c_int32(nd_level),
                                           _p(_i32(node_offsets)), _p(_i32(node_vertices))))

    def write_csv(self, path, rows):
        """pipeline.cpp:193-205 write_csv; rows = dicts with BenchRow fields."""
        k = len(rows)
        inp = (C.c_char_p * max(k, 1))(*[r["input"].encode() for r in rows])
        meth = (C.c_char_p * max(k, 1))(*[r["method"].encode() for r in rows])
        ints = np.array([[r[f] for f in ("n", "nnz_A", "patch_size", "nd_level", "nnz_L", "cost")] for r in rows],
                        np.int64).reshape(-1)
        dbl = np.array([[r[f] for f in ("t_patch_ms", "t_quotient_ms", "t_etree_ms", "t_local_ms", "t_assemble_ms",
                                         "fill_ratio")] for r in rows], np.float64).reshape(-1)
        self._check(self._f("write_csv")(os.fsencode(path), C.c_int32(k), inp, meth, _p(ints), _p(dbl)))

    def validate_user_patches(self, g, assignment, patch_count):
        """patching.cpp:386-433 -> (sizes, disconnected, unused)."""
        a = _i32(assignment)
        P = max(patch_count, 1)
        sizes, dis, unu = np.zeros(P, np.int64), np.zeros(P, np.int32), np.zeros(P, np.int32)
        nd, nu = C.c_int32(), C.c_int32()
        self._check(self._f("validate_user_patches")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                                     _p(a), C.c_int32(len(a)), C.c_int32(patch_count), _p(sizes),
                                                     _p(dis), C.byref(nd), _p(unu), C.byref(nu)))
        return sizes[:patch_count].tolist(), dis[:nd.value].tolist(), unu[:nu.value].tolist()

    def run_pipeline(self, n_rows_out, mesh_path="", matrix_path="", rows=0, cols=0, patch_file="", patch_size=256,
                     nd_level=-1, seed=0, block_size=1, out_perm="", out_etree=""):
        """pipeline.cpp:57-160 run_pipeline (timing off) -> dict(perm, nnz_L, cost, method)."""
        perm = np.zeros(max(n_rows_out, 1), np.int32)
        nnz, cost = C.c_int64(), C.c_int64()
        method = C.create_string_buffer(64)
        e = lambda x: os.fsencode(str(x))
        self._check(self._f("run_pipeline")(e(mesh_path), e(matrix_path), C.c_int32(rows), C.c_int32(cols),
                                            e(patch_file), C.c_int32(patch_size), C.c_int32(nd_level),
                                            C.c_uint64(seed), C.c_int32(block_size), e(out_perm), e(out_etree),
                                            _p(perm), C.byref(nnz), C.byref(cost), method))
        return dict(perm=perm[:n_rows_out], nnz_L=nnz.value, cost=cost.value, method=method.value.decode())

    def cross_block_fill(self, g, perm, nd_level, node_offsets, node_vertices):
        """symbolic.cpp:98-119 (the pipeline self-check, pipeline.cpp:141)."""
        c = C.c_int64()
        self._check(self._f("cross_block_fill")(C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)),
                                                _p(_i32(perm)), C.c_int32(nd_level), _p(_i32(node_offsets)),
                                                _p(_i32(node_vertices)), C.byref(c)))
        return int(c.value)

    def compute_perm_schedule(self, g, nd_level, node_offsets, node_vertices, local_perm, schedule):
        """assemble.cpp:65-85 compute_perm(tree, g, schedule) with any node sequence."""
        pm, inv = np.zeros(max(g.n, 1), np.int32), np.zeros(max(g.n, 1), np.int32)
        sched = _i32(schedule)
        self._check(self._f("compute_perm_schedule")(
            C.c_int32(g.n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)), C.c_int32(nd_level), _p(_i32(node_offsets)),
            _p(_i32(node_vertices)), _p(_i32(local_perm)), _p(sched), C.c_int64(len(sched)), _p(pm), _p(inv)))
        return pm[:g.n], inv[:g.n]

    def validate_schedule(self, nd_level, sequence):
        """assemble.cpp:48-63: first violating position or None."""
        seq = _i32(sequence)
        bad = C.c_int64()
        self._check(self._f("validate_schedule")(C.c_int32(nd_level), _p(seq), C.c_int64(len(seq)), C.byref(bad)))
        return None if bad.value < 0 else bad.value

    def order_timed(self, g, patch_size=256, nd_level=-1, seed=0, mode=0, levelorder=0, threads=1):
        """ref_order: run_pipeline's ordering stages with time_stage timers (ms per stage)."""
        n = g.n
        L = nd_level if nd_level >= 0 else self.default_nd_level(n)
        nn = (1 << (L + 1)) - 1
        asg = np.zeros(max(n, 1), np.int32)
        off = np.zeros(nn + 1, np.int32)
        verts, lp = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        pm, inv = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        pc, lo = C.c_int32(), C.c_int32()
        st = (C.c_double * 5)()
        self._check(self._f("order")(C.c_int32(n), _p(_i32(g.offsets)), _p(_i32(g.neighbors)), C.c_int32(patch_size),
                                     C.c_int32(nd_level), C.c_uint64(seed), C.c_int32(mode), C.c_int32(levelorder),
                                     C.c_int32(threads), _p(asg), C.byref(pc), C.byref(lo), _p(off), _p(verts),
                                     _p(lp), _p(pm), _p(inv), st))
        return dict(assignment=asg[:n], patch_count=pc.value, nd_level=lo.value, node_offsets=off,
                    node_vertices=verts[:n], local_perm=lp[:n], perm=pm[:n], inverse=inv[:n],
                    stage_ms=list(st), ms=float(sum(st)))
