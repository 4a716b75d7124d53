"""Profile helper: stage / kernel times of C3 (10M torus) through mp_order."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

g = mp.mesh_to_graph(mp.make_torus_mesh(2000, 5000))
ctx = mp.Context(0)
for _ in range(2):
    r = mp.order(g, ctx=ctx, want_fill=False)
print({k: round(v, 1) for k, v in r.stage_ms.items()}, {k: round(v, 1) for k, v in r.kernel_ms.items()},
      "work", r.work[:16], flush=True)
