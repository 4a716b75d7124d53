"""Arbitrary node schedules (assemble.hpp:32-38), elimination_fill /
factor_etree_parents for any permutation (symbolic.hpp:23,31) and the exact
cross_block_fill value (symbolic.hpp:37), against the reference.

The schedule validator is host code behind the C ABI, so its known answers
run without a GPU; everything that plays the elimination game is -m gpu.
"""
import numpy as np
import pytest

import paper_2602_00898_b200 as mp
from oracle.oracle import Reference


def _tree(L):
    nn = (1 << (L + 1)) - 1
    return mp.EliminationTree(0, L, np.zeros(nn + 1, np.int32), np.zeros(0, np.int32))


def random_schedule(L, rng):
    """Any valid schedule: repeatedly pick a random node whose children are done
    (the reference test's generator, tests/assemble_test.cpp:17-38)."""
    nn = (1 << (L + 1)) - 1
    done = np.zeros(nn, bool)
    ready = [i for i in range(nn) if 2 * i + 1 >= nn]
    out = []
    while ready:
        i = ready.pop(int(rng.integers(len(ready))))
        done[i] = True
        out.append(i)
        if i == 0:
            continue
        par = (i - 1) // 2
        sib = 2 * par + 1 if 2 * par + 2 == i else 2 * par + 2
        if done[sib]:
            ready.append(par)
    return out


def test_validate_schedule_known_answers():  # tests/assemble_test.cpp:66-75
    t = _tree(1)
    assert mp.validate_schedule(t, [0, 1, 2]) == 0  # root too early
    assert mp.validate_schedule(t, [1, 1, 0]) == 1  # repeat
    assert mp.validate_schedule(t, [1, 7, 0]) == 1  # out of range
    assert mp.validate_schedule(t, [1, 2]) == 2  # too short
    assert mp.validate_schedule(t, []) == 0
    assert mp.validate_schedule(t, [2, 1, 0]) is None
    assert mp.schedule_nodes(2) == [3, 4, 1, 5, 6, 2, 0]  # tests/assemble_test.cpp:51-57
    assert mp.schedule_nodes(2, "levelorder") == [3, 4, 5, 6, 1, 2, 0]
    assert mp.validate_schedule(_tree(2), mp.schedule_nodes(2)) is None


def test_validate_schedule_matches_reference_on_random_sequences():
    R = Reference()
    rng = np.random.default_rng(7)
    for L in range(0, 5):
        nn = (1 << (L + 1)) - 1
        for _ in range(40):
            kind = rng.integers(3)
            if kind == 0:
                seq = random_schedule(L, rng)
            elif kind == 1:  # a valid schedule with one swap / truncation / bad id
                seq = random_schedule(L, rng)
                j = int(rng.integers(len(seq)))
                op = rng.integers(3)
                if op == 0 and len(seq) > 1:
                    k = int(rng.integers(len(seq)))
                    seq[j], seq[k] = seq[k], seq[j]
                elif op == 1:
                    seq = seq[:j]
                else:
                    seq[j] = int(rng.integers(-2, nn + 3))
            else:
                seq = rng.integers(-1, nn + 1, int(rng.integers(0, nn + 2))).tolist()
            assert mp.validate_schedule(_tree(L), seq) == R.validate_schedule(L, seq), (L, seq)


@pytest.mark.gpu
def test_compute_perm_any_schedule_matches_reference():
    """compute_perm(tree, g, schedule) for random valid schedules, and the
    reference's error for an invalid one (assemble_test.cpp:77-90, :106-126)."""
    R = Reference()
    rng = np.random.default_rng(23)
    for seed in range(4):
        g = mp.mesh_to_graph(mp.make_random_mesh(9 + 5 * seed, 11 + 3 * seed, seed))
        p = mp.compute_patches(g, 8, seed)
        L = 3
        t = mp.order_tree_nodes(mp.build_etree(g, p.assignment, p.patch_count, L), g)
        post = mp.tree_fill(g, t, "postorder")
        for _ in range(3):
            sched = random_schedule(L, rng)
            P = mp.compute_perm(t, g, sched)
            rp, ri = R.compute_perm_schedule(g, L, t.node_offsets, t.vertices, t.local_perm, sched)
            assert np.array_equal(P.perm, rp) and np.array_equal(P.inverse, ri)
            F = mp.tree_fill(g, t, sched)
            ref = R.elimination_fill(g, rp)
            assert F.nnz_L == ref["nnz_L"] == post.nnz_L  # schedule invariance (crit. 1)
            assert F.cost == ref["cost"] and np.array_equal(F.column_counts, ref["column_counts"])
            assert np.array_equal(F.parents, R.factor_etree_parents(g, rp))
            r = mp.order(g, patch_size=8, nd_level=L, seed=seed, schedule=sched)
            assert np.array_equal(r.perm.perm, rp) and r.fill.nnz_L == post.nnz_L
        with pytest.raises(ValueError, match="invalid schedule at position 0"):
            mp.compute_perm(t, g, [0] + mp.schedule_nodes(L)[:-1])
        with pytest.raises(ValueError, match="invalid schedule at position 14"):
            mp.order(g, patch_size=8, nd_level=L, schedule=mp.schedule_nodes(L)[:-1])


@pytest.mark.gpu
def test_acceptance_criterion_1_on_device():
    """acceptance_main.cpp:105-140: post-order and level-order (and random
    schedules) give identical nnz(L) on 20 random meshes + grids 3x3..17x17;
    cross_block_fill == 0 for the ordering outputs."""
    rng = np.random.default_rng(2024)
    corpus = []
    for _ in range(20):
        rows, cols = 4 + int(rng.integers(41)), 4 + int(rng.integers(41))
        while rows * cols > 2000:
            cols = 4 + int(rng.integers(41))
        corpus.append(mp.mesh_to_graph(mp.make_random_mesh(rows, cols, int(rng.integers(1 << 62)))))
    corpus += [mp.mesh_to_graph(mp.make_grid_mesh(k, k)) for k in range(3, 18)]
    for g in corpus:
        L = 1 if g.n < 100 else (2 if g.n < 900 else 3)
        target = max(2, g.n // 12)
        p = mp.compute_patches(g, target, int(rng.integers(1 << 62)))
        t = mp.order_tree_nodes(mp.build_etree(g, p.assignment, p.patch_count, L), g)
        fills = [mp.tree_fill(g, t, s).nnz_L for s in ("postorder", "levelorder", random_schedule(L, rng))]
        assert len(set(fills)) == 1
        for s in ("postorder", "levelorder"):
            assert mp.cross_block_fill(g, mp.compute_perm(t, g, s), t) == 0


@pytest.mark.gpu
def test_elimination_fill_any_permutation_matches_reference():
    R = Reference()
    rng = np.random.default_rng(5)
    for k, g in enumerate([mp.mesh_to_graph(mp.make_grid_mesh(12, 13)),
                           mp.mesh_to_graph(mp.make_random_mesh(20, 17, 3)),
                           mp.mesh_to_graph(mp.make_icosphere_mesh(6))]):
        for perm in (np.arange(g.n, dtype=np.int32), rng.permutation(g.n).astype(np.int32)):
            F = mp.elimination_fill(g, perm)
            ref = R.elimination_fill(g, perm)
            assert (F.nnz_A, F.nnz_L, F.cost) == (ref["nnz_A"], ref["nnz_L"], ref["cost"])
            assert np.array_equal(F.column_counts, ref["column_counts"])
            assert F.fill_ratio == ref["nnz_L"] / ref["nnz_A"]
            assert np.array_equal(mp.factor_etree_parents(g, perm), R.factor_etree_parents(g, perm))
    g = mp.mesh_to_graph(mp.make_grid_mesh(4, 4))
    with pytest.raises(ValueError, match="bijection"):
        mp.elimination_fill(g, np.zeros(g.n, np.int32))
    with pytest.raises(ValueError, match="does not match"):
        mp.elimination_fill(g, np.arange(3, dtype=np.int32))


@pytest.mark.gpu
def test_cross_block_fill_known_answers_and_reference():
    cyc = mp.AdjacencyGraph(4, np.array([0, 2, 4, 6, 8], np.int32),
                            np.array([1, 3, 0, 2, 1, 3, 0, 2], np.int32))  # symbolic_test.cpp:104-129
    bad = mp.EliminationTree(4, 1, np.array([0, 0, 2, 4], np.int32), np.array([0, 1, 2, 3], np.int32))
    assert mp.cross_block_fill(cyc, np.arange(4, dtype=np.int32), bad) == 3
    good = mp.EliminationTree(4, 1, np.array([0, 2, 3, 4], np.int32), np.array([0, 2, 1, 3], np.int32))
    assert mp.cross_block_fill(cyc, np.array([1, 3, 0, 2], np.int32), good) == 0
    R = Reference()
    rng = np.random.default_rng(11)
    for seed in range(3):
        g = mp.mesh_to_graph(mp.make_random_mesh(14, 15, seed))
        p = mp.compute_patches(g, 10, seed)
        t = mp.build_etree(g, p.assignment, p.patch_count, 2)
        for perm in (rng.permutation(g.n).astype(np.int32), np.arange(g.n, dtype=np.int32)):
            assert mp.cross_block_fill(g, perm, t) == R.cross_block_fill(g, perm, 2, t.node_offsets, t.vertices)
