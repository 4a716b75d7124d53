"""Profile helper: stage / kernel times of C2 (1M icosphere) through mp_order (MP_PROFILE=1 adds per-level marks)."""
import sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2602_00898_b200 as mp
g = mp.mesh_to_graph(mp.make_icosphere_mesh(316))
ctx = mp.Context(0)
for _ in range(3):
    r = mp.order(g, ctx=ctx, want_fill=False)
print(r.stage_ms, r.kernel_ms, flush=True)
