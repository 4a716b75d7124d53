"""Probe: C3 FPS time vs the cluster / grid-mode radius threshold (MP_TUNE_FPS_GRID_RADIUS)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

g = mp.mesh_to_graph(mp.make_torus_mesh(2000, 5000))
base = None
for gr in [0, 120, 80, 250]:
    ctx = mp.Context(0)
    if gr:
        ctx.set_tuning("fps_grid_radius", gr)
    for _ in range(2):
        r = mp.order(g, ctx=ctx, want_fill=False)
    sha = hash(r.patch.assignment.tobytes())
    base = base if base is not None else sha
    print(gr, round(r.kernel_ms["fps"], 1), "same patches" if sha == base else "DIFFERENT", r.work[4:8], flush=True)
