"""Profile helper: FPS kernel time of the C2 icosphere under context tunings."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

f = int(sys.argv[1]) if len(sys.argv) > 1 else 316
g = mp.mesh_to_graph(mp.make_icosphere_mesh(f))
base = None
import json
tunes = json.loads(sys.argv[2]) if len(sys.argv) > 2 else [{}, {"fps_cluster": 8}, {"fps_grid_radius": 100},
                                                         {"fps_grid_radius": 400}]
for tune in tunes:
    ctx = mp.Context(0)
    for k, v in tune.items():
        ctx.set_tuning(k, v)
    ts = []
    for _ in range(3):
        r = mp.compute_patches(g, 256, 0, ctx=ctx) if False else mp.order(g, ctx=ctx, want_fill=False)
        ts.append(r.kernel_ms["fps"])
    same = base is None or np.array_equal(base, r.perm.perm)
    base = r.perm.perm if base is None else base
    print(tune, "same" if same else "DIFF", [round(t, 2) for t in ts], round(r.stage_ms["patch"], 2),
          [int(x) for x in r.work[4:16]], flush=True)
    ctx.close()
