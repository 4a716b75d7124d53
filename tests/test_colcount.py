"""The etree + column-count fill (csrc/colcount.cu) against the reference's
elimination game (symbolic.cpp:33-45 elimination_fill, :82-96
factor_etree_parents) and against the device game (fill_algorithm 'game').

Covers the cases the fast path treats specially: several connected pieces
per subtree (child roots), levelorder and random schedules (node position
ranges not nested), empty tree nodes, rows with more than 32 lower
neighbours (the O(d^2) branch), and a caller tree whose separators leak (the
entry point falls back to the game)."""
import numpy as np
import pytest

import paper_2602_00898_b200 as mp
from oracle.oracle import Reference

from test_schedules_and_fill import random_schedule

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctxs():
    fast = mp.Context(0)
    game = mp.Context(0)
    game.set_fill_algorithm("game")
    yield fast, game
    fast.close()
    game.close()


def _graphs():
    out = [
        ("grid", mp.mesh_to_graph(mp.make_grid_mesh(70, 53))),
        ("random", mp.mesh_to_graph(mp.make_random_mesh(60, 80, 11))),
        ("torus", mp.mesh_to_graph(mp.make_torus_mesh(40, 90))),
        ("ico", mp.mesh_to_graph(mp.make_icosphere_mesh(30))),
    ]
    a = mp.make_grid_mesh(30, 41)
    b = mp.make_random_mesh(25, 33, 5)
    c = mp.make_grid_mesh(3, 3)
    tris = np.concatenate([a.triangles, b.triangles + a.vertex_count,
                           c.triangles + a.vertex_count + b.vertex_count])
    out.append(("multi", mp.mesh_to_graph(mp.TriangleMesh(a.vertex_count + b.vertex_count + c.vertex_count, tris))))
    return out


def _check(R, g, res):
    ref = R.elimination_fill(g, res.perm.perm)
    assert res.fill.nnz_L == ref["nnz_L"]
    assert res.fill.cost == ref["cost"]
    assert np.array_equal(res.fill.column_counts, ref["column_counts"])
    assert np.array_equal(res.fill.parents, R.factor_etree_parents(g, res.perm.perm))


@pytest.mark.parametrize("L", [0, 1, 3, 6])
@pytest.mark.parametrize("schedule", ["postorder", "levelorder"])
def test_fast_fill_matches_reference_and_game(ctxs, L, schedule):
    fast, game = ctxs
    R = Reference()
    for name, g in _graphs():
        r1 = mp.order(g, patch_size=64, nd_level=L, schedule=schedule, ctx=fast)
        r2 = mp.order(g, patch_size=64, nd_level=L, schedule=schedule, ctx=game)
        assert np.array_equal(r1.perm.perm, r2.perm.perm), name
        _check(R, g, r1)
        assert np.array_equal(r1.fill.column_counts, r2.fill.column_counts), name
        assert np.array_equal(r1.fill.parents, r2.fill.parents), name


def test_fast_fill_random_schedules(ctxs):
    fast, _ = ctxs
    R = Reference()
    rng = np.random.default_rng(3)
    for name, g in _graphs()[:3]:
        L = 4
        res = mp.order(g, patch_size=48, nd_level=L, ctx=fast)
        for _ in range(4):
            sched = random_schedule(L, rng)
            f = mp.tree_fill(g, res.tree, sched, ctx=fast)
            pm = mp.compute_perm(res.tree, g, sched, ctx=fast)
            ref = R.elimination_fill(g, pm.perm)
            assert f.nnz_L == ref["nnz_L"], name
            assert np.array_equal(f.column_counts, ref["column_counts"]), name
            assert np.array_equal(f.parents, R.factor_etree_parents(g, pm.perm)), name


def _expand(g, b):
    """Block-expanded pattern (every vertex -> b rows coupled to its own and its
    neighbours' rows), the elasticity-style layout of SURVEY C5."""
    rows, offs = [], [0]
    for v in range(g.n):
        blocks = np.sort(np.concatenate([[v], g.neighbors[g.offsets[v]:g.offsets[v + 1]]]))
        cols = (blocks[:, None] * b + np.arange(b)[None, :]).ravel()
        for i in range(b):
            r = v * b + i
            row = cols[cols != r]
            rows.append(row)
            offs.append(offs[-1] + len(row))
    return mp.AdjacencyGraph(g.n * b, np.asarray(offs, np.int32), np.concatenate(rows).astype(np.int32))


def test_fast_fill_wide_rows(ctxs):
    """3x3 / 12x12 block patterns: rows with more than 32 lower neighbours."""
    fast, _ = ctxs
    R = Reference()
    base = mp.mesh_to_graph(mp.make_grid_mesh(14, 17))
    for b in (3, 12):
        g = _expand(base, b)
        res = mp.order(g, patch_size=96, nd_level=3, ctx=fast)
        _check(R, g, res)


def test_fast_fill_more_levels_than_vertices(ctxs):
    fast, game = ctxs
    R = Reference()
    g = mp.mesh_to_graph(mp.make_grid_mesh(9, 7))
    for L in (5, 8):
        r1 = mp.order(g, patch_size=4, nd_level=L, ctx=fast)
        _check(R, g, r1)


def test_leaky_tree_falls_back_to_game(ctxs):
    """A caller tree whose nodes are not separated (contiguous vertex-id ranges):
    tree_fill must still equal the reference's elimination_fill."""
    fast, _ = ctxs
    R = Reference()
    g = mp.mesh_to_graph(mp.make_grid_mesh(20, 20))
    L = 2
    nn = (1 << (L + 1)) - 1
    verts = np.arange(g.n, dtype=np.int32)
    bounds = np.linspace(0, g.n, nn + 1).astype(np.int32)
    lp = np.concatenate([np.arange(bounds[i + 1] - bounds[i], dtype=np.int32) for i in range(nn)])
    tree = mp.EliminationTree(g.n, L, bounds, verts, lp)
    assert mp.tree_separation_violations(g, tree, ctx=fast) > 0
    f = mp.tree_fill(g, tree, "postorder", ctx=fast)
    pm = mp.compute_perm(tree, g, "postorder", ctx=fast)
    ref = R.elimination_fill(g, pm.perm)
    assert f.nnz_L == ref["nnz_L"]
    assert np.array_equal(f.column_counts, ref["column_counts"])
    assert np.array_equal(f.parents, R.factor_etree_parents(g, pm.perm))
