"""TEST INFRASTRUCTURE ONLY — synthetic meshes built without the product library.

The reference arm of bench.py and the golden generator must not load
libmeshperm_b200.so, so the BASELINE inputs are rebuilt here:

* grid R x C       : make_grid_mesh (reference pipeline.cpp:38-55), via the
                     reference core itself (ref_make_grid_mesh);
* random R x C, s  : tests/test_support.hpp:66-86 random_mesh, the reference's
                     own generator (ref_random_mesh, std::mt19937_64);
* torus R x C      : SURVEY.md Appendix C (cells split like make_grid_mesh,
                     indices mod R / mod C), numpy;
* icosphere f      : SURVEY.md Appendix C numbering, numpy.

The CSR then comes from the reference's mesh_to_graph (graph.cpp:63-75).
tests/test_oracle.py checks every generator against the product's.
"""
from __future__ import annotations

import ctypes as C
import hashlib

import numpy as np

ICO_FACES = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4],
                      [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                      [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)


def torus_triangles(rows: int, cols: int) -> np.ndarray:
    r, c = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    r1, c1 = (r + 1) % rows, (c + 1) % cols
    a, b, d, e = r * cols + c, r * cols + c1, r1 * cols + c, r1 * cols + c1
    t = np.stack([a, b, d, b, e, d], -1).reshape(-1, 3)
    return t.astype(np.int32)


def icosphere_triangles(f: int) -> tuple[int, np.ndarray]:
    edges = sorted({(min(x, y), max(x, y)) for fc in ICO_FACES.tolist() for x, y in
                    ((fc[0], fc[1]), (fc[1], fc[2]), (fc[2], fc[0]))})
    eidx = {e: k for k, e in enumerate(edges)}

    def edge_points(a, b, steps):  # vertex ids at `steps` (array) from a towards b
        steps = np.asarray(steps)
        lo, hi = min(a, b), max(a, b)
        s = steps if a == lo else f - steps
        out = 12 + eidx[(lo, hi)] * (f - 1) + (s - 1)
        out = np.where(steps == 0, a, out)
        return np.where(steps == f, b, out)

    nv = 10 * f * f + 2
    nxt = 12 + 30 * (f - 1)
    tris = []
    ii, jj = np.meshgrid(np.arange(f + 1), np.arange(f + 1), indexing="ij")
    inside = (ii + jj) <= f
    interior = inside & (ii > 0) & (jj > 0) & (ii + jj < f)
    n_int = int(interior.sum())
    for a, b, c in ICO_FACES.tolist():
        G = np.full((f + 1, f + 1), -1, np.int64)
        # face-interior ids, i-major then j (the row-major order of the mask)
        G[interior] = nxt + np.arange(n_int)
        nxt += n_int
        G[:, 0] = edge_points(a, b, np.arange(f + 1))          # j == 0
        G[0, :] = edge_points(a, c, np.arange(f + 1))          # i == 0
        i = np.arange(1, f)
        G[i, f - i] = edge_points(c, b, i)                      # i + j == f
        G[f, 0] = b
        G[0, f] = c
        ti, tj = np.nonzero((ii + jj) < f)                      # up triangles, i-major
        up = np.stack([G[ti, tj], G[ti + 1, tj], G[ti, tj + 1]], -1)
        down_ok = (ti + tj + 1) < f
        dn = np.stack([G[ti + 1, tj], G[ti + 1, tj + 1], G[ti, tj + 1]], -1)
        # interleave: each up triangle is followed by its down triangle when it exists
        order = np.concatenate([up[:, None, :], dn[:, None, :]], 1).reshape(-1, 3)
        keep = np.stack([np.ones_like(down_ok), down_ok], 1).reshape(-1)
        tris.append(order[keep])
    assert nxt == nv
    return nv, np.concatenate(tris).astype(np.int32)


def mesh(kind: str, arg, R=None) -> tuple[int, np.ndarray]:
    """(vertex_count, triangles) of a BASELINE input, product library not loaded."""
    from .oracle import Reference
    R = R or Reference()
    if kind == "icosphere":
        return icosphere_triangles(int(arg))
    if kind == "torus":
        rows, cols = arg
        return rows * cols, torus_triangles(rows, cols)
    if kind == "grid":
        rows, cols = (arg, arg) if np.isscalar(arg) else arg
        return rows * cols, R.make_grid_mesh(rows, cols)
    if kind == "random":
        rows, cols, seed = arg
        return rows * cols, R.random_mesh(rows, cols, seed)
    raise ValueError(kind)


def graph(kind: str, arg, R=None):
    """(n, offsets, neighbors) built by the reference's mesh_to_graph."""
    from .oracle import Reference
    R = R or Reference()
    nv, tris = mesh(kind, arg, R)
    off, nbr = R.mesh_to_graph(nv, tris)
    return nv, off, nbr


def csr_digest(offsets, neighbors) -> str:
    h = hashlib.sha256(np.ascontiguousarray(offsets, np.int32).tobytes())
    h.update(np.ascontiguousarray(neighbors, np.int32).tobytes())
    return h.hexdigest()[:16]


__all__ = ["torus_triangles", "icosphere_triangles", "mesh", "graph", "csr_digest", "C"]
