"""Generate the golden fixtures from the REFERENCE itself (run in the build container).

Uses oracle/_ref/libmeshperm_ref.so (the unmodified reference core compiled by
oracle/Makefile from /root/reference) on inputs built by our generators:

* small.npz       — full stage outputs for a corpus of small graphs
                    (assignment, tree, local orders, perm, column counts, parents)
* bench_golden.json — scalar goldens + sha256 digests for the BASELINE configs
                    (c1 grid 64x64, ico158 C4 frame, c2 icosphere f=316)

    python tests/golden/make_golden.py [--big]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import paper_2602_00898_b200 as mp  # noqa: E402  (generators + host CSR build only)
from oracle.oracle import Reference  # noqa: E402

HERE = Path(__file__).resolve().parent

# name -> (graph builder, patch_size, nd_level, mode, levelorder)
SMALL = {
    "path4": (lambda: csr_from_edges(4, [(0, 1), (1, 2), (2, 3)]), 2, 1, 0, 0),
    "grid4x4": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(4, 4)), 4, 2, 0, 0),
    "grid12x9": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(12, 9)), 8, 2, 0, 0),
    "grid30": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), 40, -1, 0, 0),
    "grid30_exact": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), 40, 3, 1, 0),
    "grid30_natural": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), 40, 3, 2, 0),
    "grid30_level": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), 40, 3, 0, 1),
    "grid30_single": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(30, 30)), 1, 4, 0, 0),
    "rand40x50": (lambda: mp.mesh_to_graph(mp.make_random_mesh(40, 50, 7)), 32, -1, 0, 0),
    "torus30x40": (lambda: mp.mesh_to_graph(mp.make_torus_mesh(30, 40)), 50, -1, 0, 0),
    "ico12": (lambda: mp.mesh_to_graph(mp.make_icosphere_mesh(12)), 64, 3, 0, 0),
    "two_grids": (lambda: disjoint(mp.mesh_to_graph(mp.make_grid_mesh(20, 20)),
                                   mp.mesh_to_graph(mp.make_grid_mesh(7, 9))), 30, 3, 0, 0),
    "grid64": (lambda: mp.mesh_to_graph(mp.make_grid_mesh(64, 64)), 256, -1, 0, 0),
}


def csr_from_edges(n, edges):
    adj = [set() for _ in range(n)]
    for u, v in edges:
        if u != v:
            adj[u].add(v)
            adj[v].add(u)
    off = np.zeros(n + 1, np.int32)
    nbr = []
    for v in range(n):
        nb = sorted(adj[v])
        nbr += nb
        off[v + 1] = off[v] + len(nb)
    return mp.AdjacencyGraph(n, off, np.array(nbr, np.int32))


def disjoint(a, b):
    off = np.concatenate([a.offsets, a.offsets[-1] + b.offsets[1:]]).astype(np.int32)
    nbr = np.concatenate([a.neighbors, b.neighbors + a.n]).astype(np.int32)
    return mp.AdjacencyGraph(a.n + b.n, off, nbr)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def run_case(R, g, patch, L, mode, levelorder, threads=8):
    r = R.order(g, patch_size=patch, nd_level=L, seed=0, mode=mode, levelorder=levelorder, threads=threads)
    f = R.elimination_fill(g, r["perm"])
    par = R.factor_etree_parents(g, r["perm"])
    r.update(column_counts=f["column_counts"], nnz_L=f["nnz_L"], cost=f["cost"], nnz_A=f["nnz_A"], parents=par)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the 1M-vertex C2 golden (~1 min)")
    ap.add_argument("--c5", action="store_true", help="only the 2M-vertex C5 golden (3x3 blocks)")
    ap.add_argument("--c3", action="store_true", help="only the 10M-vertex C3 torus golden (~15 min)")
    ap.add_argument("--c4", action="store_true", help="only the 64 C4 frames random_mesh(500,500,seed=f)")
    args = ap.parse_args()
    R = Reference()
    if args.c5:
        return make_c5(R)
    if args.c4:
        return make_c4(R)
    if args.c3:
        return make_big(R, "c3", lambda: mp.mesh_to_graph(mp.make_torus_mesh(2000, 5000)))
    arrays = {}
    for name, (build, patch, L, mode, lo) in SMALL.items():
        g = build()
        r = run_case(R, g, patch, L, mode, lo)
        pre = name + "."
        arrays.update({pre + "offsets": g.offsets, pre + "neighbors": g.neighbors,
                       pre + "params": np.array([patch, L, mode, lo, r["nd_level"], r["patch_count"]], np.int64),
                       pre + "assignment": r["assignment"], pre + "node_offsets": r["node_offsets"],
                       pre + "node_vertices": r["node_vertices"], pre + "local_perm": r["local_perm"],
                       pre + "perm": r["perm"], pre + "inverse": r["inverse"],
                       pre + "column_counts": r["column_counts"], pre + "parents": r["parents"],
                       pre + "scalars": np.array([r["nnz_A"], r["nnz_L"], r["cost"]], np.int64)})
        print(f"{name}: n={g.n} P={r['patch_count']} L={r['nd_level']} nnz_L={r['nnz_L']}")
    np.savez_compressed(HERE / "small.npz", **arrays)

    gold_path = HERE / "bench_golden.json"
    gold = json.loads(gold_path.read_text()) if gold_path.exists() else {}
    big = [("c1", lambda: mp.mesh_to_graph(mp.make_grid_mesh(64, 64))),
           ("ico158", lambda: mp.mesh_to_graph(mp.make_icosphere_mesh(158)))]
    if args.big:
        big.append(("c2", lambda: mp.mesh_to_graph(mp.make_icosphere_mesh(316))))
    for name, build in big:
        gold[name] = big_entry(R, build)
        print(name, gold[name])
    gold_path.write_text(json.dumps(gold, indent=1) + "\n")


def make_big(R, name, build):
    gold_path = HERE / "bench_golden.json"
    gold = json.loads(gold_path.read_text())
    gold[name] = big_entry(R, build)
    print(name, gold[name])
    gold_path.write_text(json.dumps(gold, indent=1) + "\n")


def big_entry(R, build):
    g = build()
    t0 = time.time()
    r = run_case(R, g, 256, -1, 0, 0, threads=16)
    off = r["node_offsets"]
    return {"n": g.n, "edges": g.edge_count(), "patch_count": r["patch_count"], "nd_level": r["nd_level"],
            "root_separator": int(off[1] - off[0]), "nnz_A": r["nnz_A"], "nnz_L": r["nnz_L"],
            "cost": r["cost"], "sha_assignment": digest(r["assignment"]),
            "sha_node_offsets": digest(off), "sha_node_vertices": digest(r["node_vertices"]),
            "sha_local_perm": digest(r["local_perm"]), "sha_perm": digest(r["perm"]),
            "sha_column_counts": digest(r["column_counts"]), "sha_parents": digest(r["parents"]),
            "reference_s": round(time.time() - t0, 1)}


def make_c5(R, b=3):
    """configs[4]: icosphere f=447 with 3x3 blocks.  The reference orders the
    base graph and expand_blocks (graph.cpp:96-128) maps vertex v to rows
    b*v..b*v+b-1; the expanded factor's column counts follow from the base
    ones (row b*v+t of a dense block column: b*c_v - t), the identity that
    tests/test_gpu_parity.py::test_block_expansion_closed_form checks against
    the elimination game on the explicitly expanded graph."""
    g = mp.mesh_to_graph(mp.make_icosphere_mesh(447))
    t0 = time.time()
    r = run_case(R, g, 256, -1, 0, 0, threads=16)
    cc = r["column_counts"].astype(np.int64)
    cols = (b * cc[:, None] - np.arange(b)[None, :]).reshape(-1)
    pb = (b * r["perm"].astype(np.int64)[:, None] + np.arange(b)[None, :]).reshape(-1).astype(np.int32)
    # expanded factor etree: inside a block row b*k+t -> b*k+t+1, the block's
    # last row -> the first row of the parent block (or -1)
    par = r["parents"].astype(np.int64)
    parb = (b * np.arange(g.n, dtype=np.int64)[:, None] + np.arange(b)[None, :] + 1)
    parb[:, b - 1] = np.where(par < 0, -1, b * par)
    parb = parb.reshape(-1).astype(np.int32)
    gold_path = HERE / "bench_golden.json"
    gold = json.loads(gold_path.read_text())
    gold["c5"] = {"n": g.n, "edges": g.edge_count(), "block_size": b, "patch_count": r["patch_count"],
                  "nd_level": r["nd_level"], "base_nnz_L": r["nnz_L"], "sha_base_perm": digest(r["perm"]),
                  "nnz_A": int(b * b * r["nnz_A"]),
                  "nnz_L": int(cols.sum()), "cost": int((cols * cols).sum()), "sha_perm": digest(pb),
                  "sha_base_column_counts": digest(r["column_counts"]), "sha_base_parents": digest(r["parents"]),
                  "sha_column_counts": digest(cols), "sha_parents": digest(parb),
                  "reference_s": round(time.time() - t0, 1)}
    print("c5", gold["c5"])
    gold_path.write_text(json.dumps(gold, indent=1) + "\n")


def make_c4(R, frames=64, threads=None):
    """configs[3]: 64 frames random_mesh(500, 500, seed=f) (the reference's own
    generator, tests/test_support.hpp:66-86), each ordered, filled and
    etree'd by the reference core; frames run concurrently (one per core)."""
    import concurrent.futures as cf
    import os
    from oracle import meshgen
    threads = threads or os.cpu_count()

    def one(f):
        n, off, nbr = meshgen.graph("random", (500, 500, f), R)
        g = mp.AdjacencyGraph(n, off, nbr)
        r = run_case(R, g, 256, -1, 0, 0, threads=1)
        return {"frame": f, "n": n, "sha_csr": meshgen.csr_digest(off, nbr), "patch_count": r["patch_count"],
                "nnz_L": r["nnz_L"], "cost": r["cost"], "sha_perm": digest(r["perm"]),
                "sha_column_counts": digest(r["column_counts"]), "sha_parents": digest(r["parents"])}

    t0 = time.time()
    with cf.ThreadPoolExecutor(threads) as ex:
        rows = list(ex.map(one, range(frames)))
    gold_path = HERE / "bench_golden.json"
    gold = json.loads(gold_path.read_text())
    gold["c4"] = {"frames": rows, "reference_s": round(time.time() - t0, 1), "threads": threads}
    print("c4", rows[:2], gold["c4"]["reference_s"])
    gold_path.write_text(json.dumps(gold, indent=1) + "\n")


if __name__ == "__main__":
    main()
