"""Profile helper: three device CSR builds of the C2 icosphere (for an ncu launch list)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2602_00898_b200 as mp  # noqa: E402
from paper_2602_00898_b200 import api  # noqa: E402

f = int(sys.argv[1]) if len(sys.argv) > 1 else 316
mesh = mp.make_icosphere_mesh(f)
ctx = mp.default_context(0)
tri = torch.from_numpy(np.ascontiguousarray(mesh.triangles, np.int32).reshape(-1)).cuda()
n, ntri = mesh.vertex_count, tri.numel() // 3
off = torch.empty(n + 1, dtype=torch.int32, device="cuda")
nbr = torch.empty(6 * ntri, dtype=torch.int32, device="cuda")
for _ in range(3):
    nnz = api.mesh_to_graph_device_ptr(ctx, n, ntri, tri.data_ptr(), off.data_ptr(), nbr.data_ptr())
torch.cuda.synchronize()
print("nnz", nnz)
