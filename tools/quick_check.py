import sys, time
sys.path.insert(0, '.')
import numpy as np, paper_2602_00898_b200 as mp, json
for name, mesh in [("c1", mp.make_grid_mesh(64, 64)), ("ico158", mp.make_icosphere_mesh(158)), ("c2", mp.make_icosphere_mesh(316))]:
    g = mp.mesh_to_graph(mesh)
    t = time.time(); r = mp.order(g); dt = time.time() - t
    gold = json.load(open("tests/golden/bench_golden.json")).get(name)
    print(name, r.patch.patch_count, r.fill.nnz_L, gold and gold["nnz_L"], round(dt, 3), flush=True)
