"""meshperm_b200: B200-native patch-based nested-dissection permutation.

Drop-in for the ordering path of the reference meshperm library
(/root/reference/proj, arxiv 2602.00898): mesh/CSR in, patches, ND tree,
permutation, factor etree and nnz(L) out, computed by sm_100a CUDA kernels
behind the C ABI in include/meshperm_b200.h.
"""
from .api import (  # noqa: F401
    AdjacencyGraph, Context, EliminationTree, FillReport, PatchPartition, Permutation, PipelineResult,
    QuotientGraph, TriangleMesh, build_etree, build_quotient, compute_patches, compute_perm, default_context,
    default_nd_level, enforce_connectivity, make_grid_mesh, make_icosphere_mesh, make_random_mesh,
    make_torus_mesh, mesh_to_graph, mesh_to_graph_device, pattern_to_graph_device, lift_patches, run_baseline,
    BASELINES, PatchReport, validate_user_patches, order, order_batch, order_device, order_subtrees, order_tree_nodes, tree_fill, tree_separation_violations,
    elimination_fill, factor_etree_parents, cross_block_fill, validate_schedule, schedule_nodes,
    Comm, order_sharded,
)
from .formats import (  # noqa: F401
    BenchRow, bench_row, csv_header, run_baselines, write_csv, parse_matrix_market, parse_mesh, parse_obj, parse_off, read_patch_file, read_permutation, write_etree,
    write_permutation,
)
from .pipeline import PipelineRun, RunConfig, default_input_id, run_pipeline  # noqa: F401,E402
