"""Profile helper: one C4 frame (random_mesh(500, 500, seed=f)) ordered alone,
and the batch of 16 frames over 1, 2, 4 contexts: stage / kernel times."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402
from paper_2602_00898_b200 import batch  # noqa: E402

frames = [mp.mesh_to_graph(mp.make_random_mesh(500, 500, seed=f)) for f in range(32)]
ctx = mp.Context(0)
for _ in range(3):
    r = mp.order(frames[0], ctx=ctx, want_fill=True)
print("alone", {k: round(v, 2) for k, v in r.stage_ms.items()}, {k: round(v, 2) for k, v in r.kernel_ms.items()},
      "launches", r.kernel_launches, "work", r.work[:8], flush=True)
ctx.close()
import torch  # noqa: E402
import json  # noqa: E402
tunes = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [{}]
plan = [(w, t) for t in tunes for w in ((4, 6, 8) if len(sys.argv) > 1 else (1, 2, 4, 6))]
for workers, tune in plan:
    pool = batch.FramePool(0, workers)
    for c in pool.ctx:
        for k, v in tune.items():
            c.set_tuning(k, v)
    pool.order_all(frames[:workers])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = pool.order_all(frames)
    base = base if "base" in dir() else [x.perm.perm for x in res]
    same = all((x.perm.perm == b).all() for x, b in zip(res, base))
    t1 = time.perf_counter()
    print("workers", workers, tune, "32 frames wall ms", round(1e3 * (t1 - t0), 1), "same" if same else "DIFF",
          "mean frame stage sum", round(sum(sum(x.stage_ms.values()) for x in res) / len(res), 2), flush=True)
    pool.close()
