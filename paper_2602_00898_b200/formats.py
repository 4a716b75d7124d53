"""On-disk formats, mirroring core/include/meshperm/io.hpp.

Thin wrappers over the host C++ readers/writers in csrc/mesh_io.cpp (exported
through the C ABI as mp_read_mesh, mp_read_matrix_market, ...).  Same names,
accepted syntax, error texts and written bytes as the reference: its
std::runtime_error surfaces as MeshpermError (a RuntimeError) carrying the
reference's "path:line: message", validate_mesh's std::invalid_argument as
ValueError.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from ._lib import MpBenchRow, check, lib
from .api import (AdjacencyGraph, EliminationTree, PatchPartition, Permutation, PipelineResult, TriangleMesh,
                  _i32, _ptr)

_FORMAT = {"auto": 0, "off": 1, "obj": 2}


def _path(p) -> bytes:
    return os.fsencode(p)


def _read_mesh(path, fmt: str) -> TriangleMesh:
    nv, nt = C.c_int32(), C.c_int64()
    check(lib().mp_read_mesh(_path(path), _FORMAT[fmt], C.byref(nv), C.byref(nt), C.c_void_p(0)))
    tris = np.zeros((nt.value, 3), np.int32)
    if nt.value:
        check(lib().mp_read_mesh(_path(path), _FORMAT[fmt], C.byref(nv), C.byref(nt), _ptr(tris)))
    return TriangleMesh(int(nv.value), tris)


def parse_off(path) -> TriangleMesh:  # io.hpp:15
    return _read_mesh(path, "off")


def parse_obj(path) -> TriangleMesh:  # io.hpp:19
    return _read_mesh(path, "obj")


def parse_mesh(path) -> TriangleMesh:  # io.hpp:22 (.off / .obj by extension)
    return _read_mesh(path, "auto")


def parse_matrix_market(path) -> tuple[int, np.ndarray, np.ndarray]:  # io.hpp:27
    """The SparsePattern as (n, rows, cols): 0-based, symmetrised, sorted, unique."""
    n, nnz = C.c_int32(), C.c_int64()
    check(lib().mp_read_matrix_market(_path(path), C.byref(n), C.byref(nnz), C.c_void_p(0), C.c_void_p(0)))
    rows, cols = np.zeros(nnz.value, np.int32), np.zeros(nnz.value, np.int32)
    if nnz.value:
        check(lib().mp_read_matrix_market(_path(path), C.byref(n), C.byref(nnz), _ptr(rows), _ptr(cols)))
    return int(n.value), rows, cols


def read_patch_file(path, n: int) -> PatchPartition:  # io.hpp:30
    a = np.zeros(max(n, 1), np.int32)
    pc = C.c_int32()
    check(lib().mp_read_patch_file(_path(path), n, _ptr(a), C.byref(pc)))
    return PatchPartition(a[:n], int(pc.value))


def write_permutation(perm, path) -> None:  # io.hpp:33
    p = _i32(perm.perm if isinstance(perm, Permutation) else perm)
    check(lib().mp_write_permutation(_path(path), len(p), _ptr(p)))


def read_permutation(path) -> np.ndarray:  # io.hpp:34
    n = C.c_int32()
    check(lib().mp_read_permutation(_path(path), C.byref(n), C.c_void_p(0)))
    p = np.zeros(max(n.value, 1), np.int32)
    check(lib().mp_read_permutation(_path(path), C.byref(n), _ptr(p)))
    return p[:n.value]


def write_etree(tree: EliminationTree, path) -> None:  # io.hpp:37
    off, verts = _i32(tree.node_offsets), _i32(tree.vertices)
    check(lib().mp_write_etree(_path(path), int(tree.nd_level), _ptr(off), _ptr(verts)))


# ---------------------------------------------------------------- bench CSV
@dataclass
class BenchRow:  # pipeline.hpp:39-54
    input: str = ""
    n: int = 0
    nnz_A: int = 0
    method: str = ""
    patch_size: int = 0
    nd_level: int = 0
    t_patch_ms: float = 0.0
    t_quotient_ms: float = 0.0
    t_etree_ms: float = 0.0
    t_local_ms: float = 0.0
    t_assemble_ms: float = 0.0
    nnz_L: int = 0
    fill_ratio: float = 0.0
    cost: int = 0


def csv_header() -> str:  # pipeline.cpp:188-191
    return lib().mp_csv_header().decode()


def write_csv(rows, path) -> None:  # pipeline.cpp:193-205 (to a file)
    rows = list(rows)
    arr = (MpBenchRow * max(len(rows), 1))()
    for i, r in enumerate(rows):
        vals = dict(vars(r))
        vals["input"], vals["method"] = r.input.encode(), r.method.encode()
        for k, v in vals.items():
            setattr(arr[i], k, v)
    check(lib().mp_write_csv(_path(path), arr, len(rows)))


def bench_row(result: PipelineResult, g: AdjacencyGraph, input: str, method: str | None = None) -> BenchRow:
    """The BenchRow run_pipeline fills (pipeline.cpp:88-148): device stage
    times, n / nnz_A of the measured graph, method "ours-<patch size>"."""
    st = result.stage_ms
    fill = result.fill
    n = len(result.perm.perm)
    return BenchRow(input, n, fill.nnz_A if fill else n + int(g.offsets[-1]),
                    method or f"ours-{result.patch.target_size}", result.patch.target_size, result.tree.nd_level,
                    st["patch"], st["quotient"], st["etree"], st["local"], st["assemble"],
                    fill.nnz_L if fill else 0, fill.fill_ratio if fill else 0.0, fill.cost if fill else 0)


def run_baselines(g: AdjacencyGraph, names, input: str = "graph", ctx=None, **kw) -> list[BenchRow]:
    """run_baselines (pipeline.cpp:162-186): one row per baseline, `md` reported
    as "md-only"; unknown names raise ValueError like the reference."""
    from .api import BASELINES, run_baseline
    rows = []
    for name in names:
        if name not in BASELINES:
            raise ValueError("unknown baseline: " + name)
        r = run_baseline(g, name, ctx=ctx, **kw)
        rows.append(bench_row(r, g, input, "md-only" if name == "md" else name))
    return rows
