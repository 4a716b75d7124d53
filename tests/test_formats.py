"""On-disk formats: csrc/mesh_io.cpp against the reference's
core/src/io.cpp.

The first half restates the reference's own io_test.cpp cases (known answers);
the second half is differential: every file in a corpus of valid and malformed
inputs goes through both the product reader and the reference (compiled into
oracle/_ref, test infrastructure only) and must give the same result or the same
error text.  Host-only code: these run without a GPU.
"""
import os

import numpy as np
import pytest

from oracle.oracle import REFERENCE_SO, Reference

import paper_2602_00898_b200 as mp
from paper_2602_00898_b200._lib import MeshpermError

needs_ref = pytest.mark.skipif(not REFERENCE_SO.exists(), reason="reference oracle not built here")


@pytest.fixture
def put(tmp_path):
    def _put(name, text):
        p = tmp_path / name
        p.write_bytes(text.encode() if isinstance(text, str) else text)
        return str(p)
    return _put


def edges(tris):
    e = set()
    for a, b, c in np.asarray(tris).reshape(-1, 3):
        e |= {(min(a, b), max(a, b)), (min(b, c), max(b, c)), (min(a, c), max(a, c))}
    return e


# ---------------------------------------------------------------- io_test.cpp
def test_parse_off_reads_vertices_faces_comments(put):  # io_test.cpp:39-52
    m = mp.parse_off(put("square.off", "OFF\n# a unit square\n4 2 0\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n3 0 1 2\n3 0 2 3\n"))
    assert m.vertex_count == 4 and len(m.triangles) == 2
    e = edges(m.triangles)
    assert (0, 2) in e and (1, 3) not in e


def test_parse_off_fan_triangulates(put):  # io_test.cpp:54-63
    m = mp.parse_off(put("quadface.off", "OFF\n4 1 0\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n4 0 1 2 3\n"))
    assert m.triangles.tolist() == [[0, 1, 2], [0, 2, 3]]


def test_parse_off_errors_carry_line(put):  # io_test.cpp:65-81
    with pytest.raises(MeshpermError, match=":1:"):
        mp.parse_off(put("bad1.off", "OFZ\n3 1 0\n"))
    with pytest.raises(MeshpermError):
        mp.parse_off(put("bad2.off", "OFF\n3 1 0\n0 0 0\n"))
    with pytest.raises(MeshpermError, match=":6:"):
        mp.parse_off(put("bad3.off", "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 5\n"))
    with pytest.raises(MeshpermError):
        mp.parse_off(put("bad4.off", "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n2 0 1\n"))


def test_parse_obj_slashes_and_quads(put):  # io_test.cpp:83-96
    m = mp.parse_obj(put("patch.obj", "# comment\nv 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nvt 0 0\nvn 0 0 1\n"
                                      "usemtl none\nf 1/1/1 2/2/1 3/3/1 4/4/1\n"))
    assert m.vertex_count == 4
    assert m.triangles.tolist() == [[0, 1, 2], [0, 2, 3]]


def test_parse_obj_out_of_range(put):  # io_test.cpp:98-102
    with pytest.raises(MeshpermError, match=":4:"):
        mp.parse_obj(put("oob.obj", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 9\n"))


def test_parse_mesh_dispatch(put):  # io_test.cpp:104-108
    assert mp.parse_mesh(put("tri.OFF", "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n")).vertex_count == 3
    with pytest.raises(MeshpermError, match="unsupported mesh format"):
        mp.parse_mesh(put("mesh.stl", "solid x\n"))


def test_matrix_market_symmetric(put):  # io_test.cpp:110-123
    n, r, c = mp.parse_matrix_market(put("path3.mtx", "%%MatrixMarket matrix coordinate pattern symmetric\n"
                                                      "% a path on three vertices\n3 3 5\n1 1\n2 2\n3 3\n2 1\n3 2\n"))
    assert n == 3
    off = {(a, b) for a, b in zip(r, c) if a != b}
    assert off == {(0, 1), (1, 0), (1, 2), (2, 1)}


def test_matrix_market_general_symmetrizes(put):  # io_test.cpp:125-133
    n, r, c = mp.parse_matrix_market(put("gen.mtx", "%%MatrixMarket matrix coordinate real general\n"
                                                    "2 2 3\n1 2 0.5\n2 1 0.5\n1 1 3.0\n"))
    assert list(zip(r.tolist(), c.tolist())) == [(0, 0), (0, 1), (1, 0)]


def test_matrix_market_rejects(put):  # io_test.cpp:135-159
    with pytest.raises(MeshpermError, match="square"):
        mp.parse_matrix_market(put("rect.mtx", "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1.0\n"))
    with pytest.raises(MeshpermError):
        mp.parse_matrix_market(put("arr.mtx", "%%MatrixMarket matrix array real general\n"))
    with pytest.raises(MeshpermError):
        mp.parse_matrix_market(put("nob.mtx", "3 3 0\n"))
    with pytest.raises(MeshpermError):
        mp.parse_matrix_market(put("eof.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 1.0\n"))
    with pytest.raises(MeshpermError, match=":3:"):
        mp.parse_matrix_market(put("oob.mtx", "%%MatrixMarket matrix coordinate real symmetric\n3 3 1\n4 1 1.0\n"))


def test_read_patch_file_count(put):  # io_test.cpp:161-169
    path = put("patches.txt", "0\n0\n1\n1\n")
    p = mp.read_patch_file(path, 4)
    assert p.patch_count == 2 and p.assignment.tolist() == [0, 0, 1, 1]
    with pytest.raises(MeshpermError, match="expected 5 patch ids, found 4"):
        mp.read_patch_file(path, 5)
    with pytest.raises(MeshpermError, match="nonnegative"):
        mp.read_patch_file(put("neg.txt", "0\n-1\n"), 2)


def test_permutation_round_trip(tmp_path):  # io_test.cpp:171-177
    path = tmp_path / "perm.txt"
    mp.write_permutation(mp.Permutation(np.array([2, 0, 1, 3], np.int32), np.array([1, 2, 0, 3], np.int32)), path)
    assert path.read_text() == "2\n0\n1\n3\n"
    assert mp.read_permutation(path).tolist() == [2, 0, 1, 3]


def test_etree_file_format(tmp_path):  # io_test.cpp:179-193
    tree = mp.EliminationTree(3, 1, np.array([0, 1, 2, 3], np.int32), np.array([1, 0, 2], np.int32))
    path = tmp_path / "tree.txt"
    mp.write_etree(tree, path)
    assert path.read_text() == "0 0 1 1\n1 1 1 0\n2 1 1 2\n"


def test_open_errors(tmp_path):
    missing = str(tmp_path / "nope.off")
    with pytest.raises(MeshpermError, match="^cannot open " + missing + "$"):
        mp.parse_off(missing)
    bad = str(tmp_path / "no_dir" / "p.txt")
    with pytest.raises(MeshpermError, match="^cannot open " + bad + " for writing$"):
        mp.write_permutation([0], bad)


# ------------------------------------------------------------ differential
OFF_CASES = [
    "", "# only a comment\n", "OFF", "OFF\n", "OFF 3\n", "OFZ\n", "off\n3 1 0\n",
    "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n",
    "OFF 3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n",
    "OFF 3 1\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2",  # no trailing newline
    "OFF\r\n3 1 0\r\n0 0 0\r\n1 0 0\r\n0 1 0\r\n3 0 1 2\r\n",
    "OFF\n\n  # c\n\t3\t1 0 # counts\n0 0 0\n\n1 0 0 1 1\n0 1 0\n3 0 1 2 9 9\n",
    "OFF\n3\n", "OFF\n-1 0\n", "OFF\n3 -2\n", "OFF\n3x 1\n", "OFF\n3 1\n0 0\n", "OFF\n3 1\n0 0 x\n",
    "OFF\n3 1\n0 0 1e400\n1 0 0\n0 1 0\n3 0 1 2\n", "OFF\n3 1\n0 0 1e-400\n1 0 0\n0 1 0\n3 0 1 2\n",
    "OFF\n3 1\nnan inf -inf\n+1 0x1p3 .5\n0 1 0\n3 0 1 2\n", "OFF\n3 1\n1.5e3 2. -.25\n1 0 0\n0 1 0\n3 0 1 2\n",
    "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n3 0 1 1\n", "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n3 0 1 -1\n",
    "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n3 0 1 0x2\n", "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2.0\n",
    "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n+3 +0 +1 +2\n", "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n99 0 1 2\n",
    "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n", "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n\n# x\n",
    "OFF\n3 1\n0 0 0\n1 0 0\n0 1 0\n3 0 1 99999999999999999999\n",
    "OFF\n0 0 0\n", "OFF\n5 2 0\n" + "0 0 0\n" * 5 + "5 0 1 2 3 4\n3 4 3 2\n",
    "OFF\n4 1 0\n" + "0 0 0\n" * 4 + "4 0 1 2 0\n",  # fan creates a repeated corner
    "OFF\n3 1 0\n0\v0\f0\n1 0 0\n0 1 0\n3 0 1 2\n",
]

OBJ_CASES = [
    "", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n", "f 1 2 3\nv 0 0 0\nv 1 0 0\nv 0 1 0\n",
    "v 0 0\n", "v a 0 0\n", "v 0 0 0 1\nv 1 0 0\nv 0 1 0\nf 3 2 1\n", "v 0 0 0\nf 1 2\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1/2 2//3 3/1/1\n", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf /1 2 3\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 0 1 2\n", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf -1 2 3\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 1 2\n", "v 0 0 0\nv 1 0 0\nv 0 1 0\nF 1 2 3\nvt 0\nvn 0 0 1\ng x\n",
    "v 0 0 0 # c\nv 1 0 0\nv 0 1 0\n# f 1 2 9\nf 1 2 3 # tail\n", "v 0 0 0\r\nv 1 0 0\r\nv 0 1 0\r\nf 1 2 3\r\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nv 1 1 0\nv 2 2 0\nf 1 2 3 4 5\nf 5 4 9\nf 1 2 x\n",
    "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3x\n",
]

MM_CASES = [
    "", "\n", "3 3 0\n", "%%MatrixMarket matrix coordinate pattern symmetric\n",
    "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 0\n",
    "%%matrixmarket MATRIX Coordinate Pattern SYMMETRIC\n3 3 2\n2 1\n3 2\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 0\n", "%%MatrixMarket matrix coordinate real hermitian\n",
    "%%MatrixMarket matrix array real general\n", "%%MatrixMarket matrix coordinate real\n",
    "%%MatrixMarket matrix coordinate integer general\n% c\n\n  % indented\n3 3 3\n\n1 2 7\n% mid\n3 1 -2\n2 2 1\n",
    "%%MatrixMarket matrix coordinate real general\n3 3\n", "%%MatrixMarket matrix coordinate real general\n3 3 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n3 4 0\n", "%%MatrixMarket matrix coordinate real general\n-1 -1 0\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 -1\n", "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 1\n0 1 1\n", "%%MatrixMarket matrix coordinate real general\n3 3 1\n1\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 x 1\n", "%%MatrixMarket matrix coordinate real general\n3 3 1\n# 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 2\n1 2\n2 1\n3 3\n",
    "%%MatrixMarket matrix coordinate pattern general\r\n2 2 1\r\n2 1\r\n",
    "%%MatrixMarket matrix coordinate pattern general\n0 0 0\n",
    "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 1\n9 9\n",  # extra lines ignored
]

PATCH_CASES = ["", "0\n0\n1\n1\n", "0 0 1 1\n", "0 # a\n0\n\n1 1\n", "0\n-1\n0\n0\n", "0\n1.0\n1\n1\n",
               "3\n3\n3\n3\n", "0\n0\n1\n", "0\n0\n1\n1\n2\n", "7 0 0 1"]

PERM_CASES = ["", "2\n0\n1\n3\n", "2 0 1 3\n", "# c\n2\n\n0 # x\n1\n3", "-5\n99\n", "1\nx\n", "1\r\n2\r\n"]


def _same_error(ours, theirs):
    kind, _, msg = theirs.partition(": ")
    assert str(ours) == msg
    assert isinstance(ours, ValueError) == (kind == "invalid_argument")


def _diff(ours_fn, theirs_fn):
    try:
        theirs = theirs_fn()
    except ValueError as e:  # the reference raised
        with pytest.raises((MeshpermError, ValueError)) as ei:
            ours_fn()
        _same_error(ei.value, str(e))
        return None
    return ours_fn(), theirs


@needs_ref
@pytest.mark.parametrize("i", range(len(OFF_CASES)))
@pytest.mark.parametrize("fmt", ["off", "auto"])
def test_off_matches_reference(put, i, fmt):
    path = put(f"c{i}.off", OFF_CASES[i])
    r = _diff(lambda: mp.parse_off(path) if fmt == "off" else mp.parse_mesh(path),
              lambda: Reference().parse_mesh(path, 1 if fmt == "off" else 0))
    if r:
        m, (nv, tris) = r
        assert m.vertex_count == nv and np.array_equal(m.triangles, tris)


@needs_ref
@pytest.mark.parametrize("i", range(len(OBJ_CASES)))
def test_obj_matches_reference(put, i):
    path = put(f"c{i}.Obj", OBJ_CASES[i])
    for fmt in (2, 0):
        r = _diff(lambda: mp.parse_obj(path) if fmt == 2 else mp.parse_mesh(path),
                  lambda: Reference().parse_mesh(path, fmt))
        if r:
            m, (nv, tris) = r
            assert m.vertex_count == nv and np.array_equal(m.triangles, tris)


@needs_ref
@pytest.mark.parametrize("i", range(len(MM_CASES)))
def test_matrix_market_matches_reference(put, i):
    path = put(f"c{i}.mtx", MM_CASES[i])
    r = _diff(lambda: mp.parse_matrix_market(path), lambda: Reference().parse_matrix_market(path))
    if r:
        (n, rows, cols), (n2, rows2, cols2) = r
        assert n == n2 and np.array_equal(rows, rows2) and np.array_equal(cols, cols2)


@needs_ref
@pytest.mark.parametrize("i", range(len(PATCH_CASES)))
def test_patch_file_matches_reference(put, i):
    path = put(f"p{i}.txt", PATCH_CASES[i])
    r = _diff(lambda: mp.read_patch_file(path, 4), lambda: Reference().read_patch_file(path, 4))
    if r:
        p, (a, pc) = r
        assert p.patch_count == pc and np.array_equal(p.assignment, a)


@needs_ref
@pytest.mark.parametrize("i", range(len(PERM_CASES)))
def test_read_permutation_matches_reference(put, i):
    path = put(f"q{i}.txt", PERM_CASES[i])
    r = _diff(lambda: mp.read_permutation(path), lambda: Reference().read_permutation(path))
    if r:
        assert np.array_equal(r[0], r[1])


@needs_ref
def test_large_files_match_reference(tmp_path):
    """A 40K-vertex mesh written as OFF (with quads and comments) and OBJ, and its
    matrix pattern as MatrixMarket; both readers agree on every index."""
    rng = np.random.default_rng(7)
    m = mp.make_random_mesh(200, 200, 3)
    tris = np.asarray(m.triangles)
    lines = ["OFF", f"{m.vertex_count} {len(tris)} 0"]
    lines += [f"{x:.3f} {y:.3e} 0" for x, y in rng.random((m.vertex_count, 2))]
    lines += [f"3 {a} {b} {c}" + (" # t" if k % 97 == 0 else "") for k, (a, b, c) in enumerate(tris)]
    off = tmp_path / "big.off"
    off.write_text("\n".join(lines) + "\n")
    obj = tmp_path / "big.obj"
    obj.write_text("".join(f"v {k} 0 1\n" for k in range(m.vertex_count))
                   + "".join(f"f {a + 1}/1 {b + 1}//2 {c + 1}\n" for a, b, c in tris))
    R = Reference()
    for p in (off, obj):
        got = mp.parse_mesh(p)
        nv, ref = R.parse_mesh(str(p))
        assert got.vertex_count == nv == m.vertex_count
        assert np.array_equal(got.triangles, ref) and np.array_equal(got.triangles, tris)
    g = mp.mesh_to_graph(m)
    rows = np.repeat(np.arange(g.n), np.diff(g.offsets))
    keep = rows > g.neighbors  # lower triangle only, as symmetric storage
    mtx = tmp_path / "big.mtx"
    mtx.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n"
                   + f"{g.n} {g.n} {int(keep.sum()) + g.n}\n"
                   + "".join(f"{i + 1} {i + 1}\n" for i in range(g.n))
                   + "".join(f"{a + 1} {b + 1}\n" for a, b in zip(rows[keep], g.neighbors[keep])))
    n, r1, c1 = mp.parse_matrix_market(mtx)
    n2, r2, c2 = R.parse_matrix_market(str(mtx))
    assert n == n2 == g.n and np.array_equal(r1, r2) and np.array_equal(c1, c2)
    assert len(r1) == g.offsets[-1] + g.n


@needs_ref
@pytest.mark.parametrize("L", [0, 1, 3])
def test_writers_byte_identical(tmp_path, L):
    rng = np.random.default_rng(L)
    n = 500
    perm = rng.permutation(n).astype(np.int32)
    mp.write_permutation(perm, tmp_path / "a.txt")
    Reference().write_permutation(str(tmp_path / "b.txt"), perm)
    assert (tmp_path / "a.txt").read_bytes() == (tmp_path / "b.txt").read_bytes()
    assert np.array_equal(mp.read_permutation(tmp_path / "a.txt"), perm)
    nodes = (1 << (L + 1)) - 1
    cuts = np.sort(rng.integers(0, n + 1, nodes - 1))
    node_offsets = np.concatenate([[0], cuts, [n]]).astype(np.int32)
    tree = mp.EliminationTree(n, L, node_offsets, perm)
    mp.write_etree(tree, tmp_path / "t1.txt")
    Reference().write_etree(str(tmp_path / "t2.txt"), n, L, node_offsets, perm)
    assert (tmp_path / "t1.txt").read_bytes() == (tmp_path / "t2.txt").read_bytes()


# ------------------------------------------------------------------ bench CSV
def _rows(k, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(k):
        out.append(mp.BenchRow(
            input=["grid-64x64", "mesh.off", "a,b"][i % 3], n=int(rng.integers(0, 10**7)),
            nnz_A=int(rng.integers(0, 10**9)), method=["ours-256", "natural", "md-only", "nd-vertex"][i % 4],
            patch_size=int(rng.integers(1, 1000)), nd_level=int(rng.integers(0, 12)),
            t_patch_ms=float(rng.choice([0.0, 0.0005, 0.0015, 2.5e-4, 1234.56789, 1e12])),
            t_quotient_ms=float(rng.random() * 10), t_etree_ms=float(rng.random() * 1e4), t_local_ms=0.0125,
            t_assemble_ms=float(rng.random()), nnz_L=int(rng.integers(0, 2**40)),
            fill_ratio=float(rng.random() * 30), cost=int(rng.integers(0, 2**62))))
    return out


@needs_ref
@pytest.mark.parametrize("k", [0, 1, 7])
def test_csv_byte_identical(tmp_path, k):
    """pipeline.cpp:188-205: header and %.3f / %.6f formatting, byte for byte."""
    rows = _rows(k, k)
    mp.write_csv(rows, tmp_path / "a.csv")
    Reference().write_csv(str(tmp_path / "b.csv"), [vars(r) for r in rows])
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
    assert (tmp_path / "a.csv").read_text().splitlines()[0] == mp.csv_header()


def test_run_baselines_unknown_name():
    with pytest.raises(ValueError, match="unknown baseline: foo"):
        mp.run_baselines(None, ["foo"])
