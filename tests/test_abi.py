"""CPU: the C-ABI library loads and exports every entry point of
include/meshperm_b200.h; host-side helpers (generators, CSR build, tree
arithmetic) behave like the reference.  No compute call needs a GPU here."""
import ctypes as C
import re
import subprocess

from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

import paper_2602_00898_b200 as mp
from paper_2602_00898_b200 import _lib


def declared_functions():
    text = (ROOT / "include" / "meshperm_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mp_\w+)", out))
    assert set(names) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_nd_level():
    assert b"sm_100a" in _lib.lib().mp_version()
    assert [mp.default_nd_level(n) for n in (1, 511, 1024, 4096, 90000, 1 << 20)] == [0, 0, 1, 3, 7, 8]


def test_grid_mesh_matches_reference_layout():
    m = mp.make_grid_mesh(3, 4)  # pipeline.cpp:38-55
    assert m.vertex_count == 12 and len(m.triangles) == 2 * 2 * 3
    assert m.triangles[0].tolist() == [0, 1, 4] and m.triangles[1].tolist() == [1, 5, 4]
    with pytest.raises(ValueError):
        mp.make_grid_mesh(1, 5)


def test_icosphere_and_torus_shapes():
    for f in (1, 2, 5, 16):
        g = mp.mesh_to_graph(mp.make_icosphere_mesh(f))
        deg = np.diff(g.offsets)
        assert g.n == 10 * f * f + 2 and g.edge_count() == 30 * f * f
        assert (deg == 5).sum() == 12 and (deg[deg != 5] == 6).all()
    g = mp.mesh_to_graph(mp.make_torus_mesh(5, 7))
    assert g.n == 35 and (np.diff(g.offsets) == 6).all()


def test_mesh_to_graph_invariants_and_errors():
    g = mp.mesh_to_graph(mp.make_random_mesh(9, 8, 5))
    for v in range(g.n):
        nb = g.neighbors_of(v)
        assert (np.diff(nb) > 0).all() and v not in nb
        for w in nb:
            assert v in g.neighbors_of(w)
    bad = mp.TriangleMesh(3, np.array([[0, 1, 1]], np.int32))
    with pytest.raises(ValueError, match="repeated corners"):
        mp.mesh_to_graph(bad)
    bad = mp.TriangleMesh(3, np.array([[0, 1, 7]], np.int32))
    with pytest.raises(ValueError, match="outside"):
        mp.mesh_to_graph(bad)


def test_result_struct_layout():
    # mp_result as declared: 8 pointers + scalars + float[6] + int64 + float[6] + int64[16]
    assert C.sizeof(_lib.MpResult) >= 8 * 8 + 8 + 3 * 8 + 8 + 24 + 8 + 24 + 128
    assert [f[0] for f in _lib.MpConfig._fields_] == ["patch_size", "nd_level", "seed", "local_mode", "schedule",
                                                      "block_size", "want_fill", "user_patches", "user_patch_count",
                                                      "schedule_nodes", "schedule_len"]


def test_struct_offsets_match_header(tmp_path):
    """ctypes mirrors of mp_csr / mp_config / mp_result / mp_bench_row have the
    offsets and sizes the C compiler gives the header's declarations."""
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    structs = {"mp_csr": _lib.MpCsr, "mp_config": _lib.MpConfig, "mp_result": _lib.MpResult,
               "mp_bench_row": _lib.MpBenchRow, "mp_comm": _lib.MpComm}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "meshperm_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for f in py._fields_:
            lines.append(f'  printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "abi"
    subprocess.run(["gcc", "-I", str(Path(__file__).resolve().parents[1] / "include"), str(src), "-o", str(exe)],
                   check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                         check=True).stdout.splitlines())
    for cname, py in structs.items():
        assert int(got[f"{cname} sizeof"]) == C.sizeof(py), cname
        for f in py._fields_:
            assert int(got[f"{cname} {f[0]}"]) == getattr(py, f[0]).offset, (cname, f[0])
