import sys; sys.path.insert(0,'.')
import numpy as np, paper_2602_00898_b200 as mp
from oracle.oracle import Restatement
R = Restatement()
def graph(n, edges):
    adj = [set() for _ in range(n)]
    for u, v in edges: adj[u].add(v), adj[v].add(u)
    off = np.zeros(n + 1, np.int32); nbr = []
    for v in range(n):
        nbr += sorted(adj[v]); off[v + 1] = len(nbr)
    return mp.AdjacencyGraph(n, off, np.array(nbr, np.int32))
g = graph(40, [(1, 2), (2, 3), (1, 3)] + [(v, v + 1) for v in range(10, 39)])
for patch in (1,3,8):
    o = R.compute_patches(g, patch, 0)
    try:
        p = mp.compute_patches(g, patch, 0)
        print(patch, p.patch_count, o[1], np.array_equal(p.assignment, o[0]), p.assignment.tolist(), o[0].tolist())
    except Exception as e:
        print(patch, "ERR", e)
