"""Profile helper: stage / kernel times of the C1 (64x64 grid) ordering under
different context tunings (results must not change)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

g = mp.mesh_to_graph(mp.make_grid_mesh(64, 64))
base = None
for tune in [{}, {"lloyd_blocks": 1}, {"lloyd_blocks": 4}, {"lloyd_blocks": 16}, {"fps_cluster": -1},
             {"fps_cluster": 8}]:
    ctx = mp.Context(0)
    for k, v in tune.items():
        ctx.set_tuning(k, v)
    for _ in range(3):
        r = mp.order(g, ctx=ctx, want_fill=False)
    st = {k: round(v, 3) for k, v in r.stage_ms.items()}
    km = {k: round(v, 3) for k, v in r.kernel_ms.items()}
    same = base is None or np.array_equal(base, r.perm.perm)
    base = r.perm.perm if base is None else base
    print(tune, "same" if same else "DIFF", st, km, r.kernel_launches)
    ctx.close()
