"""Profile helper: per-section wall times (MP_PROFILE=1, synchronising) of
one C1 ordering after warm-up, aggregated over the ND levels."""
import collections
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "64"
if arg.startswith("ico"):
    g = mp.mesh_to_graph(mp.make_icosphere_mesh(int(arg[3:])))
elif arg.startswith("torus"):
    g = mp.mesh_to_graph(mp.make_torus_mesh(2000, 5000))
elif arg.startswith("rand"):
    g = mp.mesh_to_graph(mp.make_random_mesh(500, 500, seed=0))
else:
    g = mp.mesh_to_graph(mp.make_grid_mesh(int(arg), int(arg)))
ctx = mp.Context(0)
for _ in range(3):
    r = mp.order(g, ctx=ctx, want_fill=False)
print({k: round(v, 3) for k, v in r.stage_ms.items()}, {k: round(v, 3) for k, v in r.kernel_ms.items()})
os.environ["MP_PROFILE"] = "1"
r = mp.order(g, ctx=ctx, want_fill=False)
