"""ctypes binding of the C ABI in include/meshperm_b200.h.

Loads the in-tree libmeshperm_b200.so and fails loudly when it is missing:
there is no CPU fallback for the ordering path.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmeshperm_b200.so"

MP_OK, MP_EINVAL, MP_ECUDA, MP_ENOMEM, MP_ELOGIC, MP_EIO = 0, 1, 2, 3, 4, 5
LOCAL_MODES = {"approx_md": 0, "exact_md": 1, "natural": 2}
SCHEDULES = {"postorder": 0, "levelorder": 1}

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)


class MpCsr(C.Structure):
    _fields_ = [("n", C.c_int32), ("offsets", C.c_void_p), ("neighbors", C.c_void_p), ("on_device", C.c_int32)]


class MpConfig(C.Structure):
    _fields_ = [
        ("patch_size", C.c_int32),
        ("nd_level", C.c_int32),
        ("seed", C.c_uint64),
        ("local_mode", C.c_int32),
        ("schedule", C.c_int32),
        ("block_size", C.c_int32),
        ("want_fill", C.c_int32),
        ("user_patches", C.c_void_p),
        ("user_patch_count", C.c_int32),
        ("schedule_nodes", C.c_void_p),
        ("schedule_len", C.c_int64),
    ]


class MpResult(C.Structure):
    _fields_ = [
        ("on_device", C.c_int32),
        ("patch_of", C.c_void_p),
        ("tree_node_offsets", C.c_void_p),
        ("tree_vertices", C.c_void_p),
        ("tree_local_perm", C.c_void_p),
        ("perm", C.c_void_p),
        ("inverse", C.c_void_p),
        ("etree_parent", C.c_void_p),
        ("column_counts", C.c_void_p),
        ("patch_count", C.c_int32),
        ("nd_level", C.c_int32),
        ("nnz_A", C.c_int64),
        ("nnz_L", C.c_int64),
        ("cost", C.c_int64),
        ("fill_ratio", C.c_double),
        ("stage_ms", C.c_float * 6),
        ("kernel_launches", C.c_int64),
        ("kernel_ms", C.c_float * 6),
        ("work", C.c_int64 * 16),
    ]


# int allgather(void* user, const void* send, void* recv, int64_t bytes, void* stream)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class MpComm(C.Structure):  # mp_comm (include/meshperm_b200.h)
    _fields_ = [
        ("rank", C.c_int32),
        ("world", C.c_int32),
        ("device_buffers", C.c_int32),
        ("allgather", C.c_void_p),
        ("user", C.c_void_p),
    ]


class MpBenchRow(C.Structure):  # pipeline.hpp:39-54 BenchRow
    _fields_ = [
        ("input", C.c_char_p),
        ("n", C.c_int64),
        ("nnz_A", C.c_int64),
        ("method", C.c_char_p),
        ("patch_size", C.c_int32),
        ("nd_level", C.c_int32),
        ("t_patch_ms", C.c_double),
        ("t_quotient_ms", C.c_double),
        ("t_etree_ms", C.c_double),
        ("t_local_ms", C.c_double),
        ("t_assemble_ms", C.c_double),
        ("nnz_L", C.c_int64),
        ("fill_ratio", C.c_double),
        ("cost", C.c_int64),
    ]


# (name, restype, argtypes) of every exported entry point; tests check that the
# library exports exactly these.
SIGNATURES = [
    ("mp_last_error", C.c_char_p, []),
    ("mp_version", C.c_char_p, []),
    ("mp_context_create", C.c_int, [C.POINTER(C.c_void_p), C.c_int32]),
    ("mp_context_destroy", None, [C.c_void_p]),
    ("mp_context_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("mp_order", C.c_int, [C.c_void_p, C.POINTER(MpCsr), C.POINTER(MpConfig), C.POINTER(MpResult)]),
    ("mp_order_batch", C.c_int,
     [C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.POINTER(MpCsr), C.POINTER(MpConfig), C.POINTER(MpResult),
      C.c_void_p]),
    ("mp_default_nd_level", C.c_int32, [C.c_int32]),
    ("mp_compute_patches", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_int32, C.c_uint64, C.c_void_p, C.c_int32, i32p]),
    ("mp_enforce_connectivity", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, i32p]),
    ("mp_validate_user_patches", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, i32p, C.c_void_p, i32p]),
    ("mp_build_quotient", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, i64p]),
    ("mp_build_etree", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_void_p, C.c_int32, C.c_int32, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int32]),
    ("mp_order_tree_nodes", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]),
    ("mp_order_subtrees", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
      C.c_void_p, C.c_void_p, C.c_int32]),
    ("mp_compute_perm", C.c_int,
     [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
      C.c_int32]),
    ("mp_tree_fill", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
      C.c_void_p, C.c_int32, i64p, i64p, i64p, C.POINTER(C.c_double)]),
    ("mp_validate_schedule", C.c_int, [C.c_int32, C.c_void_p, C.c_int64, i64p]),
    ("mp_compute_perm_schedule", C.c_int,
     [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
      C.c_void_p, C.c_int32]),
    ("mp_tree_fill_schedule", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
      C.c_void_p, C.c_void_p, C.c_int32, i64p, i64p, i64p, C.POINTER(C.c_double)]),
    ("mp_elimination_fill", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, i64p, i64p, i64p,
      C.POINTER(C.c_double)]),
    ("mp_cross_block_fill", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, i64p]),
    ("mp_order_sharded", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.POINTER(MpConfig), C.POINTER(MpComm), C.POINTER(MpResult)]),
    ("mp_nccl_get_unique_id", C.c_int, [C.c_void_p]),
    ("mp_nccl_comm_init", C.c_int, [C.POINTER(MpComm), C.c_void_p, C.c_int32, C.c_int32, C.c_int32]),
    ("mp_nccl_comm_destroy", None, [C.POINTER(MpComm)]),
    ("mp_grid_mesh_triangles", C.c_int64, [C.c_int32, C.c_int32]),
    ("mp_make_grid_mesh", C.c_int, [C.c_int32, C.c_int32, C.c_void_p]),
    ("mp_make_random_mesh", C.c_int, [C.c_int32, C.c_int32, C.c_uint64, C.c_void_p]),
    ("mp_torus_mesh_triangles", C.c_int64, [C.c_int32, C.c_int32]),
    ("mp_make_torus_mesh", C.c_int, [C.c_int32, C.c_int32, C.c_void_p]),
    ("mp_icosphere_vertices", C.c_int64, [C.c_int32]),
    ("mp_icosphere_triangles", C.c_int64, [C.c_int32]),
    ("mp_make_icosphere_mesh", C.c_int, [C.c_int32, C.c_void_p]),
    ("mp_mesh_to_graph", C.c_int, [C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, i64p]),
    ("mp_tree_separation_check", C.c_int,
     [C.c_void_p, C.POINTER(MpCsr), C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, i64p]),
    ("mp_context_set_sm_share", C.c_int, [C.c_void_p, C.c_int32]),
    ("mp_context_set_fill_algorithm", C.c_int, [C.c_void_p, C.c_int32]),
    ("mp_context_set_tuning", C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    ("mp_pattern_to_graph_device", C.c_int,
     [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
      C.c_int32, i64p]),
    ("mp_lift_patches", C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]),
    ("mp_mesh_to_graph_device", C.c_int,
     [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, i64p]),
    ("mp_read_mesh", C.c_int, [C.c_char_p, C.c_int32, i32p, i64p, C.c_void_p]),
    ("mp_read_matrix_market", C.c_int, [C.c_char_p, i32p, i64p, C.c_void_p, C.c_void_p]),
    ("mp_read_patch_file", C.c_int, [C.c_char_p, C.c_int32, C.c_void_p, i32p]),
    ("mp_write_permutation", C.c_int, [C.c_char_p, C.c_int32, C.c_void_p]),
    ("mp_read_permutation", C.c_int, [C.c_char_p, i32p, C.c_void_p]),
    ("mp_write_etree", C.c_int, [C.c_char_p, C.c_int32, C.c_void_p, C.c_void_p]),
    ("mp_csv_header", C.c_char_p, []),
    ("mp_write_csv", C.c_int, [C.c_char_p, C.POINTER(MpBenchRow), C.c_int32]),
]

_lib = None


def lib() -> C.CDLL:
    """The loaded library (raises if the CUDA extension has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2602_00898_b200.build` "
                "(there is no CPU fallback for the ordering path)")
        l = C.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


class MeshpermError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def check(code: int) -> None:
    if code != MP_OK:
        msg = (lib().mp_last_error() or b"").decode()
        if code == MP_EINVAL:
            raise ValueError(msg)  # std::invalid_argument in the reference
        raise MeshpermError(code, msg)
