"""ctypes binding of libmsk.so (include/msk.h).  Argument marshalling only.

Every computation happens in the CUDA kernels of libmsk.so; this module has
no numerical code and no fallback: if the library cannot be loaded, or no
CUDA device is usable, the calls raise.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MSK_LIB_PATH: development override (A/B timing of alternative in-tree builds)
LIB_PATH = os.environ.get("MSK_LIB_PATH") or os.path.join(_HERE, "libmsk.so")

MSK_OK, MSK_ERR_INVALID, MSK_ERR_NOMEM, MSK_ERR_CUDA, MSK_ERR_NCCL, MSK_ERR_NOCONV, MSK_ERR_STATE = range(7)
MSK_SCHED_PRUNED = 0
MSK_SCHED_LITERAL = 1
MSK_MAX_LEVELS = 16
STATUS_NAMES = {0: "MSK_OK", 1: "MSK_ERR_INVALID", 2: "MSK_ERR_NOMEM", 3: "MSK_ERR_CUDA",
                4: "MSK_ERR_NCCL", 5: "MSK_ERR_NOCONV", 6: "MSK_ERR_STATE"}

_i32, _i64, _dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
_vp = ctypes.c_void_p


class SolveInfo(ctypes.Structure):
    _fields_ = [("L", _i32), ("jacobi_sweeps", _i32),
                ("cg_iters", _i32 * MSK_MAX_LEVELS), ("inner_iters", _i32 * MSK_MAX_LEVELS),
                ("rel_res", _dbl * MSK_MAX_LEVELS),
                ("nnz_cg", _dbl), ("nnz_gather", _dbl), ("bytes_cg", _dbl),
                ("t_cg_ms", _dbl), ("t_gather_ms", _dbl), ("t_total_ms", _dbl),
                ("t_cg_level_ms", _dbl * MSK_MAX_LEVELS), ("bytes_cg_level", _dbl * MSK_MAX_LEVELS),
                ("launches", _i32), ("kappa_est", _dbl * MSK_MAX_LEVELS)]


class HierarchyInfo(ctypes.Structure):
    _fields_ = [("d", _i32), ("L", _i32), ("k", _i32),
                ("n", _i64 * MSK_MAX_LEVELS), ("nnz_A", _i64 * MSK_MAX_LEVELS),
                ("ncells", _i64 * MSK_MAX_LEVELS),
                ("delta", _dbl * MSK_MAX_LEVELS), ("q", _dbl * MSK_MAX_LEVELS),
                ("t_create_ms", _dbl), ("t_assemble_ms", _dbl),
                ("launches_create", _i32), ("launches_assemble", _i32)]


class EvalInfo(ctypes.Structure):
    _fields_ = [("nnz", _dbl), ("t_sort_ms", _dbl), ("t_eval_ms", _dbl), ("t_total_ms", _dbl),
                ("launches", _i32)]


class MskError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load() -> ctypes.CDLL:
    """Load libmsk.so (in-tree build).  Raises if it is missing: there is no fallback."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmsk.so not built ({LIB_PATH}); run "
                          "`python -m paper_2503_04914_b200.build` (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    pp = ctypes.POINTER(_vp)
    sig = {
        "msk_ctx_create": ([ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _vp, pp], ctypes.c_int),
        "msk_ctx_destroy": ([_vp], None),
        "msk_hierarchy_create": ([_vp, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_i64), pp,
                                  ctypes.POINTER(_dbl), ctypes.POINTER(_dbl), ctypes.c_int,
                                  ctypes.c_uint32, pp], ctypes.c_int),
        "msk_hierarchy_destroy": ([_vp], None),
        "msk_hierarchy_info_get": ([_vp, ctypes.POINTER(HierarchyInfo)], ctypes.c_int),
        "msk_assemble": ([_vp, _dbl, _dbl], ctypes.c_int),
        "msk_assemble_ex": ([_vp, _dbl, _dbl, _dbl, _i64], ctypes.c_int),
        "msk_set_threshold": ([_vp, _dbl], ctypes.c_int),
        "msk_solve": ([_vp, pp, _dbl, _i32, ctypes.c_uint32, pp, ctypes.POINTER(SolveInfo)], ctypes.c_int),
        "msk_evaluate": ([_vp, _i64, _vp, _vp], ctypes.c_int),
        "msk_evaluate_ex": ([_vp, _i64, _vp, _vp, ctypes.POINTER(EvalInfo)], ctypes.c_int),
        "msk_solve_multi": ([_vp, _i32, pp, _dbl, _i32, pp, _vp, ctypes.POINTER(_dbl)], ctypes.c_int),
        "msk_evaluate_multi": ([_vp, _i64, _vp, _vp], ctypes.c_int),
        "msk_m_norm": ([_vp, _i32, _dbl, _dbl, ctypes.POINTER(_dbl), ctypes.POINTER(_i32)], ctypes.c_int),
        "msk_m_norm_ex": ([_vp, _i32, _i32, _dbl, _dbl, ctypes.POINTER(_dbl), ctypes.POINTER(_i32)], ctypes.c_int),
        "msk_export_block": ([_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp], ctypes.c_int),
        "msk_export_cells": ([_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
        "msk_export_grid": ([_vp, ctypes.c_int, _vp, _vp, _vp], ctypes.c_int),
        "msk_export_factor": ([_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, ctypes.POINTER(_dbl)],
                              ctypes.c_int),
        "msk_apply_block": ([_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, ctypes.POINTER(_dbl)], ctypes.c_int),
        "msk_cg_level": ([_vp, ctypes.c_int, _vp, _vp, _dbl, _i32, ctypes.POINTER(_i32),
                          ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)], ctypes.c_int),
        "msk_nccl_unique_id": ([_vp], ctypes.c_int),
        "msk_partition_rows": ([_i64, ctypes.c_int, ctypes.POINTER(_i64)], ctypes.c_int),
        "msk_halo_plan": ([ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(_i64)] * 7, ctypes.c_int),
        "msk_last_error": ([], ctypes.c_char_p),
        "msk_version": ([], ctypes.c_char_p),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


EXPORTED = ["msk_ctx_create", "msk_ctx_destroy", "msk_hierarchy_create", "msk_hierarchy_destroy",
            "msk_hierarchy_info_get", "msk_assemble", "msk_assemble_ex", "msk_set_threshold", "msk_solve", "msk_evaluate", "msk_evaluate_ex",
            "msk_solve_multi", "msk_evaluate_multi", "msk_m_norm", "msk_m_norm_ex",
            "msk_export_block", "msk_export_factor", "msk_export_cells", "msk_export_grid", "msk_apply_block", "msk_cg_level",
            "msk_nccl_unique_id", "msk_partition_rows", "msk_halo_plan", "msk_last_error", "msk_version"]
MSK_FLAG_DIST_ALL = 1
MSK_FLAG_MATRIX_FREE = 2
MSK_FLAG_OUTPUT_LOCAL = 4


def check(status: int) -> None:
    if status != MSK_OK:
        raise MskError(status, load().msk_last_error().decode())
