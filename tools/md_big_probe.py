"""Profile helper: MD of nodes above 8K vertices (md_node_global) -- a
grid with one ND level (two ~20K leaves) and a 200x200 grid ordered as one
node -- plus C3-size leaves when asked."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402

cases = [("grid200_L0", mp.make_grid_mesh(200, 200), 0), ("grid280_L1", mp.make_grid_mesh(280, 280), 1)]
for name, m, L in cases:
    g = mp.mesh_to_graph(m)
    for _ in range(2):
        r = mp.order(g, nd_level=L, want_fill=False)
    print(name, g.n, "md ms", round(r.kernel_ms["md"], 2), "local", round(r.stage_ms["local"], 2), flush=True)
