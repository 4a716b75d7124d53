import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


GOLDEN = ROOT / "tests" / "golden"


class Case:
    def __init__(self, z, name):
        import paper_2602_00898_b200 as mp
        self.name = name
        g = lambda k: z[f"{name}.{k}"]
        self.g = mp.AdjacencyGraph(len(g("offsets")) - 1, g("offsets"), g("neighbors"))
        self.patch, self.L_arg, self.mode, self.levelorder, self.L, self.patch_count = [int(x) for x in g("params")]
        for k in ["assignment", "node_offsets", "node_vertices", "local_perm", "perm", "inverse", "column_counts",
                  "parents"]:
            setattr(self, k, g(k))
        self.nnz_A, self.nnz_L, self.cost = [int(x) for x in g("scalars")]


def golden_cases():
    z = np.load(GOLDEN / "small.npz")
    names = sorted({k.split(".")[0] for k in z.files})
    return [Case(z, n) for n in names]


@pytest.fixture(scope="session")
def cases():
    return golden_cases()
