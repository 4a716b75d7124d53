"""run_pipeline (core/include/meshperm/pipeline.hpp:17-81, core/src/pipeline.cpp:57-160).

The reference's top-level entry point, same RunConfig fields and checks:
exactly one input source (mesh file, MatrixMarket file, or a synthetic grid),
optional user patch file, block size, output files.  The graph build, the
patch validation / repair and the ordering run on the GPU (mp_mesh_to_graph_device,
mp_pattern_to_graph_device, mp_order); the readers / writers are the host
C++ of csrc/mesh_io.cpp.  The BenchRow carries device-timed stage times.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import api, formats
from ._lib import MP_ELOGIC, MeshpermError


@dataclass
class RunConfig:  # pipeline.hpp:17-37
    mesh_path: str = ""
    matrix_path: str = ""
    grid_rows: int = 0
    grid_cols: int = 0
    patch_file: str = ""
    patch_size: int = 256
    nd_level: int = -1
    schedule: str = "postorder"
    local_mode: str = "approx_md"
    block_size: int = 1
    seed: int = 0
    threads: int = 1          # accepted for parity; the device path has no host threads to set
    collect_timing: bool = True
    out_perm: str = ""
    out_etree: str = ""
    input_id: str = ""


@dataclass
class PipelineRun:  # pipeline.hpp:56-61 PipelineResult
    row: formats.BenchRow
    perm: api.Permutation
    tree: api.EliminationTree
    fill: api.FillReport
    patch: api.PatchPartition
    extra: dict = field(default_factory=dict)


def _basename(path: str) -> str:  # pipeline.cpp:23-26
    cut = max(path.rfind("/"), path.rfind("\\"))
    return path if cut < 0 else path[cut + 1:]


def default_input_id(c: RunConfig) -> str:  # pipeline.cpp:28-34
    if c.input_id:
        return c.input_id
    if c.mesh_path:
        return _basename(c.mesh_path)
    if c.matrix_path:
        return _basename(c.matrix_path)
    return f"grid-{c.grid_rows}x{c.grid_cols}"


def run_pipeline(config: RunConfig, ctx: api.Context | None = None) -> PipelineRun:
    """pipeline.cpp:57-160 on the device.  Raises ValueError for the
    reference's invalid_argument cases and MeshpermError (MP_ELOGIC) if the
    separator self-check fails."""
    c = config
    sources = bool(c.mesh_path) + bool(c.matrix_path) + (c.grid_rows > 0 or c.grid_cols > 0)
    if sources != 1:
        raise ValueError("exactly one input source must be given")
    b = c.block_size
    if b < 1:
        raise ValueError("block size must be positive")
    if c.patch_size < 1:
        raise ValueError("patch size must be positive")
    ctx = ctx or api.default_context()

    # ordering graph (one node per block) and measurement graph (one per row)
    if c.matrix_path:
        n, rows, cols = formats.parse_matrix_market(c.matrix_path)
        measure = api.pattern_to_graph_device(n, rows, cols, 1, ctx=ctx)
        ordering = api.pattern_to_graph_device(n, rows, cols, b, ctx=ctx) if b > 1 else measure
    else:
        mesh = formats.parse_mesh(c.mesh_path) if c.mesh_path else api.make_grid_mesh(c.grid_rows, c.grid_cols)
        ordering = api.mesh_to_graph_device(mesh, ctx=ctx)
        measure = None  # mp_order's fill covers expand_graph(ordering, b) exactly (closed form)

    L = c.nd_level if c.nd_level >= 0 else api.default_nd_level(ordering.n)
    user = formats.read_patch_file(c.patch_file, ordering.n) if c.patch_file else None
    kw = dict(patch_size=c.patch_size, nd_level=L, seed=c.seed, local_mode=c.local_mode, schedule=c.schedule,
              block_size=b, ctx=ctx, user_patches=user)
    if measure is None or b == 1:
        res = api.order(ordering, want_fill=True, **kw)
        fill = res.fill
        nnz_a_graph_n = ordering.n * b
    else:
        # matrix with blocks: order the compressed graph, count fill on the
        # row graph with the expanded tree (its separators still separate)
        res = api.order(ordering, want_fill=False, **kw)
        if api.tree_separation_violations(measure, res.tree, ctx=ctx) != 0:
            raise MeshpermError(MP_ELOGIC, "separator failed to disconnect its sides")
        fill = api.tree_fill(measure, res.tree, c.schedule, ctx=ctx)
        nnz_a_graph_n = measure.n

    st = res.stage_ms if c.collect_timing else dict.fromkeys(res.stage_ms, 0.0)
    row = formats.BenchRow(default_input_id(c), nnz_a_graph_n, fill.nnz_A,
                           "user-patches" if c.patch_file else f"ours-{c.patch_size}", c.patch_size, L,
                           st["patch"], st["quotient"], st["etree"], st["local"], st["assemble"],
                           fill.nnz_L, fill.fill_ratio, fill.cost)
    if c.out_perm:
        formats.write_permutation(res.perm, c.out_perm)
    if c.out_etree:
        formats.write_etree(res.tree, c.out_etree)
    return PipelineRun(row, res.perm, res.tree, fill, res.patch, {"stage_ms": res.stage_ms})
