"""Randomised parity sweep: mesh families x seeds x patch sizes x ND depths x
local modes x schedules, every output of mp_order against the reference core
(oracle/_ref, compiled from /root/reference) on the same inputs.  Sizes are kept
small enough (<= ~25K vertices) that the reference finishes in well under a
second per case."""
import numpy as np
import pytest

from oracle.oracle import Reference

import paper_2602_00898_b200 as mp

pytestmark = pytest.mark.gpu

MODES = ["approx_md", "exact_md", "natural"]
SCHED = ["postorder", "levelorder"]


def _graph(kind, rng):
    if kind == "grid":
        return mp.mesh_to_graph(mp.make_grid_mesh(int(rng.integers(5, 140)), int(rng.integers(5, 140))))
    if kind == "random":
        return mp.mesh_to_graph(mp.make_random_mesh(int(rng.integers(5, 120)), int(rng.integers(5, 120)),
                                                    int(rng.integers(0, 1 << 30))))
    if kind == "torus":
        return mp.mesh_to_graph(mp.make_torus_mesh(int(rng.integers(3, 120)), int(rng.integers(3, 120))))
    if kind == "ico":
        return mp.mesh_to_graph(mp.make_icosphere_mesh(int(rng.integers(1, 45))))
    # two disjoint meshes: several components
    a = mp.make_grid_mesh(int(rng.integers(3, 40)), int(rng.integers(3, 40)))
    b = mp.make_random_mesh(int(rng.integers(3, 40)), int(rng.integers(3, 40)), 3)
    tris = np.concatenate([a.triangles, b.triangles + a.vertex_count])
    return mp.mesh_to_graph(mp.TriangleMesh(a.vertex_count + b.vertex_count, tris))


CASES = [(k, s) for k in ["grid", "random", "torus", "ico", "multi"] for s in range(12)]


@pytest.mark.parametrize("kind,seed", CASES, ids=[f"{k}-{s}" for k, s in CASES])
def test_sweep_matches_reference(kind, seed):
    rng = np.random.default_rng(1000 * seed + len(kind))
    g = _graph(kind, rng)
    patch = int(rng.choice([4, 16, 37, 64, 128, 256]))
    L = int(rng.choice([-1, -1, 0, 1, 2, 3, 5]))
    mode = int(rng.choice([0, 0, 1, 2])) if g.n <= 6000 else 0  # exact MD only at small sizes (reference cost)
    sched = int(rng.integers(0, 2))
    pseed = int(rng.integers(0, 1 << 40))
    R = Reference()
    o = R.order(g, patch_size=patch, nd_level=L, seed=pseed, mode=mode, levelorder=sched)
    r = mp.order(g, patch_size=patch, nd_level=L, seed=pseed, local_mode=MODES[mode], schedule=SCHED[sched])
    assert r.patch.patch_count == o["patch_count"]
    assert np.array_equal(r.patch.assignment, o["assignment"])
    assert np.array_equal(r.tree.node_offsets, o["node_offsets"])
    assert np.array_equal(r.tree.vertices, o["node_vertices"])
    assert np.array_equal(r.tree.local_perm, o["local_perm"])
    assert np.array_equal(r.perm.perm, o["perm"]) and np.array_equal(r.perm.inverse, o["inverse"])
    f = R.elimination_fill(g, o["perm"])
    assert r.fill.nnz_L == f["nnz_L"] and r.fill.cost == f["cost"]
    assert np.array_equal(r.fill.column_counts, f["column_counts"])
