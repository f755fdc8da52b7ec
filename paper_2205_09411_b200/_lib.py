"""ctypes binding of libpmg_b200.so (include/pmg_b200.h).

Fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libpmg_b200.so")

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")


class LsfT(C.Structure):
    _fields_ = [
        ("shape", C.c_int32), ("cylindrical", C.c_int32), ("center", C.c_double * 3),
        ("radius", C.c_double), ("seg_a", C.c_double * 3), ("seg_b", C.c_double * 3),
        ("boundary_value", C.c_double), ("shift_p", C.c_double), ("shift_q", C.c_double),
        ("scale", C.c_double),
    ]


class StencilCfgT(C.Structure):
    _fields_ = [
        ("eps_tol", C.c_double), ("max_bracket_iters", C.c_int32), ("d_min", C.c_double),
        ("w_min", C.c_double), ("boundary_safety", C.c_double), ("thin_rescue", C.c_int32),
    ]


class MgCfgT(C.Structure):
    _fields_ = [
        ("n_down", C.c_int32), ("n_up", C.c_int32), ("coarse_rel_tol", C.c_double),
        ("coarse_max_iters", C.c_int32), ("threads", C.c_int32),
    ]


class StatsT(C.Structure):
    _fields_ = [("max_resid", C.c_double), ("l2_resid", C.c_double)]


# status codes (include/pmg_types.h)
PMG_OK = 0
PMG_ERR_INVALID_ARG = 1
PMG_ERR_CUDA = 2
PMG_ERR_COARSE_STALL = 3
PMG_ERR_NONFINITE = 4
PMG_ERR_STATE = 5
PMG_ERR_TOPOLOGY = 6

EXPORTS = [
    "pmg_b200_create", "pmg_b200_destroy", "pmg_b200_last_error", "pmg_b200_stream",
    "pmg_b200_set_mesh", "pmg_b200_set_face_bc", "pmg_b200_set_stencils",
    "pmg_b200_build_stencils", "pmg_b200_stencil_summary", "pmg_b200_get_stencils",
    "pmg_b200_set_boundary_value", "pmg_b200_upload_field", "pmg_b200_download_field",
    "pmg_b200_upload_level_field", "pmg_b200_download_level_field", "pmg_b200_solver_create",
    "pmg_b200_init", "pmg_b200_v_cycle", "pmg_b200_fmg_cycle", "pmg_b200_measure_residual",
    "pmg_b200_v_cycle_async", "pmg_b200_fmg_cycle_async", "pmg_b200_cycle_result",
    "pmg_b200_gsrb_sweep", "pmg_b200_fill_ghosts", "pmg_b200_apply_pins",
    "pmg_b200_residual_level", "pmg_b200_restrict_level", "pmg_b200_restrict_level_no_guess",
    "pmg_b200_prolong_correction", "pmg_b200_prolong_full", "pmg_b200_coarse_solve",
    "pmg_b200_set_have_guess", "pmg_b200_coarse_sizes", "pmg_b200_coarse_get",
    "pmg_b200_cycle_kernel_count", "pmg_b200_n_levels", "pmg_b200_level_size",
    "pmg_b200_synchronize", "pmg_b200_time_op", "pmg_b200_coarse_info", "pmg_b200_level_classes",
    "pmg_b200_set_owned", "pmg_b200_level_field_ptr", "pmg_b200_restrict_only", "pmg_b200_fas_level",
    "pmg_b200_level_record", "pmg_b200_n_leaves", "pmg_b200_face_gradient", "pmg_b200_error_norms",
    "pmg_b200_write_dump", "pmg_b200_stage_field_async", "pmg_b200_commit_staged_field",
    "pmg_b200_set_partition", "pmg_b200_nccl_unique_id", "pmg_b200_dist_init_nccl",
    "pmg_b200_dist_local_group", "pmg_b200_dist_v_cycle", "pmg_b200_dist_v_cycle_async",
    "pmg_b200_dist_info", "pmg_b200_field_bytes", "pmg_b200_host_buffer",
    "pmg_b200_tree_create", "pmg_b200_tree_destroy", "pmg_b200_tree_last_error",
    "pmg_b200_tree_n_blocks", "pmg_b200_tree_n_levels", "pmg_b200_tree_adapt_passes",
    "pmg_b200_tree_refine_all", "pmg_b200_tree_adapt", "pmg_b200_tree_refine_by_criterion",
    "pmg_b200_tree_get", "pmg_b200_tree_level_blocks", "pmg_b200_tree_device_arrays",
    "pmg_b200_set_mesh_from_tree",
]

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise RuntimeError(
            f"libpmg_b200.so not built ({SO_PATH}); run `python -m paper_2205_09411_b200.build` "
            "-- the B200 path has no CPU fallback")
    lib = C.CDLL(SO_PATH)
    vp = C.c_void_p
    lib.pmg_b200_create.restype = vp
    lib.pmg_b200_create.argtypes = [C.c_int, C.c_int, f64p, f64p, C.c_int]
    lib.pmg_b200_destroy.argtypes = [vp]
    lib.pmg_b200_last_error.restype = C.c_char_p
    lib.pmg_b200_last_error.argtypes = [vp]
    lib.pmg_b200_stream.restype = vp
    lib.pmg_b200_stream.argtypes = [vp]
    lib.pmg_b200_set_mesh.argtypes = [vp, C.c_int, i32p, i32p, f64p, f64p, i32p, i32p, i32p, i32p]
    lib.pmg_b200_set_face_bc.argtypes = [vp, C.c_int, C.c_int, C.c_void_p]
    lib.pmg_b200_set_stencils.argtypes = [vp, i32p, i32p, i32p, f64p, f64p, f64p, f64p, i8p, u8p,
                                          i8p, i32p, C.c_int, f64p]
    lib.pmg_b200_build_stencils.argtypes = [vp, C.c_void_p, C.c_int, C.POINTER(StencilCfgT)]
    lib.pmg_b200_stencil_summary.argtypes = [vp, i32p, i32p]
    lib.pmg_b200_get_stencils.argtypes = [vp, i32p, f64p, f64p, f64p, f64p, i8p, u8p, i8p, i32p]
    lib.pmg_b200_set_boundary_value.argtypes = [vp, C.c_int, C.c_double]
    for n in ("pmg_b200_upload_field", "pmg_b200_download_field"):
        getattr(lib, n).argtypes = [vp, C.c_int, C.c_void_p, C.c_int]
    for n in ("pmg_b200_upload_level_field", "pmg_b200_download_level_field"):
        getattr(lib, n).argtypes = [vp, C.c_int, C.c_int, C.c_void_p, C.c_int]
    lib.pmg_b200_solver_create.argtypes = [vp, C.POINTER(MgCfgT)]
    for n in ("pmg_b200_init", "pmg_b200_v_cycle_async", "pmg_b200_fmg_cycle_async",
              "pmg_b200_coarse_solve", "pmg_b200_synchronize"):
        getattr(lib, n).argtypes = [vp]
    for n in ("pmg_b200_v_cycle", "pmg_b200_fmg_cycle", "pmg_b200_measure_residual",
              "pmg_b200_cycle_result"):
        getattr(lib, n).argtypes = [vp, C.POINTER(StatsT)]
    for n in ("pmg_b200_gsrb_sweep", "pmg_b200_fill_ghosts"):
        getattr(lib, n).argtypes = [vp, C.c_int, C.c_int]
    for n in ("pmg_b200_apply_pins", "pmg_b200_residual_level", "pmg_b200_restrict_level",
              "pmg_b200_restrict_level_no_guess", "pmg_b200_prolong_correction",
              "pmg_b200_prolong_full", "pmg_b200_set_have_guess", "pmg_b200_n_levels",
              "pmg_b200_cycle_kernel_count", "pmg_b200_level_size"):
        getattr(lib, n).argtypes = [vp, C.c_int]
    lib.pmg_b200_n_levels.argtypes = [vp]
    lib.pmg_b200_coarse_sizes.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                          C.POINTER(C.c_int32)]
    lib.pmg_b200_coarse_get.argtypes = [vp, i32p, i32p, f64p, f64p, f64p, i32p, i32p]
    lib.pmg_b200_level_classes.argtypes = [vp, C.c_int, i32p]
    lib.pmg_b200_time_op.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.pmg_b200_coarse_info.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_double)]
    lib.pmg_b200_set_owned.argtypes = [vp, C.c_int, C.c_void_p]
    lib.pmg_b200_level_field_ptr.argtypes = [vp, C.c_int, C.c_int]
    lib.pmg_b200_level_field_ptr.restype = C.c_void_p
    for n in ("pmg_b200_restrict_only", "pmg_b200_fas_level"):
        getattr(lib, n).argtypes = [vp, C.c_int]
    lib.pmg_b200_level_record.argtypes = [vp, C.c_int, f64p]
    lib.pmg_b200_n_leaves.argtypes = [vp]
    lib.pmg_b200_face_gradient.argtypes = [vp, C.c_int, f64p, C.c_void_p, C.c_void_p]
    lib.pmg_b200_write_dump.argtypes = [vp, C.c_int, C.c_char_p, C.c_char_p]
    lib.pmg_b200_stage_field_async.argtypes = [vp, C.c_int, C.c_int, C.c_void_p, C.c_int]
    lib.pmg_b200_commit_staged_field.argtypes = [vp]
    lib.pmg_b200_error_norms.argtypes = [vp, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double)]
    lib.pmg_b200_set_partition.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_void_p]
    lib.pmg_b200_nccl_unique_id.argtypes = [C.c_void_p]
    lib.pmg_b200_dist_init_nccl.argtypes = [vp, C.c_void_p]
    lib.pmg_b200_dist_local_group.argtypes = [C.c_int, C.POINTER(vp)]
    lib.pmg_b200_dist_v_cycle.argtypes = [vp, C.POINTER(StatsT)]
    lib.pmg_b200_dist_v_cycle_async.argtypes = [vp]
    lib.pmg_b200_dist_info.argtypes = [vp, C.POINTER(C.c_int32)]
    lib.pmg_b200_field_bytes.argtypes = [vp, C.POINTER(C.c_double)]
    lib.pmg_b200_host_buffer.argtypes = [vp, C.c_size_t]
    lib.pmg_b200_host_buffer.restype = C.c_void_p
    # the block tree on the device (csrc/tree.cu)
    lib.pmg_b200_tree_create.restype = vp
    lib.pmg_b200_tree_create.argtypes = [C.c_int, C.c_int, f64p, f64p, C.c_int]
    lib.pmg_b200_tree_destroy.argtypes = [vp]
    lib.pmg_b200_tree_last_error.restype = C.c_char_p
    lib.pmg_b200_tree_last_error.argtypes = [vp]
    for n in ("pmg_b200_tree_n_blocks", "pmg_b200_tree_n_levels", "pmg_b200_tree_adapt_passes"):
        getattr(lib, n).argtypes = [vp]
    lib.pmg_b200_tree_refine_all.argtypes = [vp, C.c_int, C.c_int]
    lib.pmg_b200_tree_adapt.argtypes = [vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
    lib.pmg_b200_tree_refine_by_criterion.argtypes = [vp, C.c_int, C.c_void_p, C.c_int, C.c_double,
                                                      C.c_double, C.c_void_p, C.c_int]
    lib.pmg_b200_tree_get.argtypes = [vp] + [C.c_void_p] * 8
    lib.pmg_b200_tree_level_blocks.argtypes = [vp, C.c_int, C.c_void_p, C.POINTER(C.c_int)]
    lib.pmg_b200_tree_device_arrays.argtypes = [vp, C.POINTER(C.c_void_p)]
    lib.pmg_b200_set_mesh_from_tree.argtypes = [vp, vp]
    _lib = lib
    return lib


class PmgError(RuntimeError):
    """Raised with the reference's exception text (std::runtime_error what())."""

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
