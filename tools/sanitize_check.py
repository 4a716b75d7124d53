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
