"""Stage-by-stage GPU vs oracle parity report (debugging aid; run on a GPU box)."""
import sys, time, traceback
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2602_00898_b200 as mp
from oracle.oracle import Restatement

R = Restatement()

def first_diff(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        return f"shape {a.shape} vs {b.shape}"
    idx = np.nonzero(a != b)[0]
    return "equal" if len(idx) == 0 else f"{len(idx)} diffs, first at {idx[0]}: {a[idx[0]]} vs {b[idx[0]]}"

def check(name, g, patch_size=256, nd_level=-1, mode="approx_md"):
    L = nd_level if nd_level >= 0 else mp.default_nd_level(g.n)
    m = {"approx_md": 0, "exact_md": 1, "natural": 2}[mode]
    print(f"== {name}: n={g.n} patch={patch_size} L={L} mode={mode}", flush=True)
    t = time.time()
    asg, pc = R.compute_patches(g, patch_size, 0)
    off, verts = R.build_etree(g, asg, pc, L)
    lp = R.order_tree_nodes(g, L, off, verts, m)
    pm, inv = R.compute_perm(g, L, off, verts, lp)
    fill = R.elimination_fill(g, pm)
    par = R.factor_etree_parents(g, pm)
    print(f"  oracle {time.time()-t:.2f}s P={pc} nnzL={fill['nnz_L']}", flush=True)
    ok = True
    try:
        p = mp.compute_patches(g, patch_size, 0)
        r = first_diff(p.assignment, asg); print(f"  patches: P {p.patch_count} vs {pc}; {r}", flush=True)
        ok &= r == "equal" and p.patch_count == pc
    except Exception:
        traceback.print_exc(); ok = False
    try:
        t2 = mp.build_etree(g, asg, pc, L)
        r1, r2 = first_diff(t2.node_offsets, off), first_diff(t2.vertices, verts)
        print(f"  etree: offsets {r1}; vertices {r2}", flush=True)
        ok &= r1 == r2 == "equal"
    except Exception:
        traceback.print_exc(); ok = False
    try:
        tr = mp.EliminationTree(g.n, L, off, verts)
        mp.order_tree_nodes(tr, g, mode)
        r = first_diff(tr.local_perm, lp); print(f"  local: {r}", flush=True); ok &= r == "equal"
        tr.local_perm = lp
        P = mp.compute_perm(tr, g)
        r = first_diff(P.perm, pm); print(f"  perm: {r}", flush=True); ok &= r == "equal"
        F = mp.tree_fill(g, tr)
        r1 = first_diff(F.column_counts, fill['column_counts']); r2 = first_diff(F.parents, par)
        print(f"  fill: nnzL {F.nnz_L} vs {fill['nnz_L']}; counts {r1}; parents {r2}", flush=True)
        ok &= r1 == r2 == "equal" and F.nnz_L == fill['nnz_L'] and F.cost == fill['cost']
    except Exception:
        traceback.print_exc(); ok = False
    try:
        res = mp.order(g, patch_size=patch_size, nd_level=nd_level, local_mode=mode)
        r = first_diff(res.perm.perm, pm)
        print(f"  order: perm {r}; nnzL {res.fill.nnz_L}; stage_ms {res.stage_ms}; launches {res.kernel_launches}", flush=True)
        ok &= r == "equal" and res.fill.nnz_L == fill['nnz_L']
    except Exception:
        traceback.print_exc(); ok = False
    print(f"  {'PASS' if ok else 'FAIL'}", flush=True)
    return ok

if __name__ == "__main__":
    cases = [
        ("grid12x9", mp.mesh_to_graph(mp.make_grid_mesh(12, 9)), dict(patch_size=8, nd_level=2)),
        ("grid64", mp.mesh_to_graph(mp.make_grid_mesh(64, 64)), {}),
        ("rand", mp.mesh_to_graph(mp.make_random_mesh(40, 50, 1)), dict(patch_size=32)),
        ("ico10", mp.mesh_to_graph(mp.make_icosphere_mesh(10)), dict(patch_size=64)),
        ("torus", mp.mesh_to_graph(mp.make_torus_mesh(30, 40)), dict(patch_size=50)),
        ("exact", mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), dict(patch_size=40, mode="exact_md")),
        ("single", mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), dict(patch_size=1)),
        ("grid300", mp.mesh_to_graph(mp.make_grid_mesh(300, 300)), {}),
    ]
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        cases.append(("ico158", mp.mesh_to_graph(mp.make_icosphere_mesh(158)), {}))
    only = [a for a in sys.argv[1:] if a != "big"]
    res = [check(n, g, **kw) for n, g, kw in cases if not only or n in only]
    print("ALL PASS" if all(res) else f"FAILURES: {res.count(False)}")
