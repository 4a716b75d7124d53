"""Profile helper: stage / kernel times of small orderings (C1 and a few
mid-size meshes) under different context tunings (results must not change)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

meshes = {
    "grid64": mp.make_grid_mesh(64, 64),
    "grid128": mp.make_grid_mesh(128, 128),
    "grid181": mp.make_grid_mesh(181, 181),
    "ico50": mp.make_icosphere_mesh(50),
    "ico100": mp.make_icosphere_mesh(100),
}
import json
tunes = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}, {"lloyd_cluster_n": -1}]
if len(sys.argv) > 2:
    meshes["ico316"] = mp.make_icosphere_mesh(316)
for name, mesh in meshes.items():
    g = mp.mesh_to_graph(mesh)
    base = None
    for tune in tunes:
        ctx = mp.Context(0)
        for k, v in tune.items():
            ctx.set_tuning(k, v)
        best = None
        for _ in range(5):
            r = mp.order(g, ctx=ctx, want_fill=False)
            tot = sum(r.stage_ms.values())
            if best is None or tot < best[0]:
                best = (tot, r)
        tot, r = best
        st = {k: round(v, 3) for k, v in r.stage_ms.items()}
        km = {k: round(v, 3) for k, v in r.kernel_ms.items()}
        same = base is None or np.array_equal(base, r.perm.perm)
        base = r.perm.perm if base is None else base
        print(name, g.n, tune, "same" if same else "DIFF", round(tot, 3), st, km, r.kernel_launches, flush=True)
        ctx.close()
