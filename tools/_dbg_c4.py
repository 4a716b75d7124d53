import sys, time, traceback
import numpy as np
sys.path.insert(0, ".")
import paper_2602_00898_b200 as mp
from oracle.oracle import Reference
R = Reference()
for seed in range(3):
    g = mp.mesh_to_graph(mp.make_random_mesh(500, 500, seed=seed))
    try:
        t = time.time(); r = mp.order(g); dt = time.time() - t
        o = R.order(g, threads=16)
        print(seed, "ok", round(dt, 3), r.patch.patch_count, o["patch_count"], np.array_equal(r.perm.perm, o["perm"]), flush=True)
    except Exception as e:
        print(seed, "ERR", e, flush=True)
        traceback.print_exc()
