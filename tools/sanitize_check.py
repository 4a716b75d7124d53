"""Small orderings for compute-sanitizer runs (memcheck / racecheck):
C1 and a random mesh, checked against the committed goldens / oracle."""
import sys
sys.path.insert(0, '.')
import json
import numpy as np
import paper_2602_00898_b200 as mp

g = mp.mesh_to_graph(mp.make_grid_mesh(64, 64))
r = mp.order(g)
assert r.fill.nnz_L == 141682, r.fill.nnz_L
g2 = mp.mesh_to_graph(mp.make_random_mesh(40, 37, 3))
r2 = mp.order(g2, patch_size=16, nd_level=4)
m = mp.mesh_to_graph_device(mp.make_grid_mesh(20, 30))
assert mp.tree_separation_violations(g2, r2.tree) == 0
# a single component above 2^15 vertices: the cluster + batched FPS kernels
g3 = mp.mesh_to_graph(mp.make_icosphere_mesh(int(sys.argv[1]) if len(sys.argv) > 1 else 60))
r3 = mp.order(g3)
print("sanitize ok", r.fill.nnz_L, r2.fill.nnz_L, m.edge_count(), g3.n, r3.patch.patch_count, r3.fill.nnz_L)
# round 2 paths: the game fill (fill algorithm 1) against the etree + counts
# fill, the fill of an arbitrary permutation, a block pattern (rows with more
# than 32 lower neighbours), and a node large enough to compact its MD pool
ctx = mp.Context(0)
ctx.set_fill_algorithm("game")
rg = mp.order(g2, patch_size=16, nd_level=4, ctx=ctx)
assert np.array_equal(rg.fill.column_counts, r2.fill.column_counts)
perm = np.random.default_rng(1).permutation(g2.n).astype(np.int32)
fe = mp.elimination_fill(g2, perm)
rows, offs = [], [0]
b = 12
g4 = mp.mesh_to_graph(mp.make_grid_mesh(12, 9))
blk_rows, blk_off = [], [0]
for v in range(g4.n):
    blocks = np.sort(np.concatenate([[v], g4.neighbors[g4.offsets[v]:g4.offsets[v + 1]]]))
    cols = (blocks[:, None] * b + np.arange(b)[None, :]).ravel()
    for i in range(b):
        row = cols[cols != v * b + i]
        blk_rows.append(row)
        blk_off.append(blk_off[-1] + len(row))
g5 = mp.AdjacencyGraph(g4.n * b, np.asarray(blk_off, np.int32), np.concatenate(blk_rows).astype(np.int32))
r5 = mp.order(g5, patch_size=64, nd_level=2)
r6 = mp.order(mp.mesh_to_graph(mp.make_grid_mesh(90, 90)), patch_size=2000, nd_level=1)
# session-d paths: 7K-vertex leaves (the compact MD layout), and the small
# mesh paths of C1 above (shared-memory FPS, one-CTA Lloyd, refine with
# shared-memory state, the shared-memory repair split)
r7 = mp.order(mp.mesh_to_graph(mp.make_grid_mesh(120, 120)), patch_size=256, nd_level=1)
print("round2 paths ok", rg.fill.nnz_L, fe.nnz_L, r5.fill.nnz_L, r6.fill.nnz_L, r7.fill.nnz_L)
# session f paths (MP_SAN_LARGE=1): the FM compact 5-byte layout with the
# prefetch helper warp (a root of ~11K patches) and md_kernel16 (one 11K-vertex
# node: 16-bit shared-memory degrees, 256-thread CTA)
import os
if os.environ.get("MP_SAN_LARGE"):
    from oracle.oracle import Reference
    g4 = mp.mesh_to_graph(mp.make_grid_mesh(150, 150))
    r4 = mp.order(g4, patch_size=2, want_fill=False)
    o4 = Reference().order(g4, patch_size=2)
    assert np.array_equal(r4.perm.perm, o4["perm"]), "fm compact"
    g5 = mp.mesh_to_graph(mp.make_grid_mesh(110, 100))
    r5 = mp.order(g5, nd_level=0, want_fill=False)
    o5 = Reference().order(g5, nd_level=0, mode=0)
    assert np.array_equal(r5.perm.perm, o5["perm"]), "md16"
    print("sanitize large ok", r4.patch.patch_count, g5.n)
