"""ctypes declarations for libaz.so (include/az.h).  Argument marshalling only.

The library is built in-tree (paper_2308_14490_b200/libaz.so, see build.py).  If it is
missing this module raises: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libaz.so")

AZ_OK = 0
AZ_WARN_SKETCH_SATURATED = 100
STATUS = {0: "AZ_OK", 1: "AZ_ERR_INVALID_ARGUMENT", 2: "AZ_ERR_OVERSAMPLING", 3: "AZ_ERR_SINGULAR_SYMBOL",
          4: "AZ_ERR_OUT_OF_MEMORY", 5: "AZ_ERR_CUDA", 6: "AZ_ERR_NOT_SUPPORTED", 7: "AZ_ERR_WORKSPACE",
          8: "AZ_ERR_NCCL",
          100: "AZ_WARN_SKETCH_SATURATED"}


class PlanDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int64), ("L", C.c_int32), ("T", C.c_double),
                ("eps", C.c_double), ("op", C.c_int32), ("row_scale", C.c_double),
                ("mask", C.c_void_p), ("n_boundary", C.c_int64), ("boundary_xy", C.c_void_p),
                ("boundary_weight", C.c_double), ("zstar_rcond", C.c_double), ("seed", C.c_uint64),
                ("k0sq", C.c_double), ("n_y", C.c_int64), ("T_y", C.c_double),
                ("boundary_coef", C.c_void_p)]


class PlanInfo(C.Structure):
    _fields_ = [("N", C.c_int64), ("M", C.c_int64), ("Mb", C.c_int64), ("sigma_max", C.c_double),
                ("sigma_min_kept", C.c_double), ("n_dropped", C.c_int64), ("zstar_norm", C.c_double)]


class SolveReport(C.Structure):
    _fields_ = [("rank_used", C.c_int64), ("probes_used", C.c_int64), ("saturated", C.c_int32),
                ("sigma_first", C.c_double), ("sigma_last_kept", C.c_double),
                ("ms_rhs", C.c_double), ("ms_sketch", C.c_double), ("ms_qr", C.c_double),
                ("ms_svd", C.c_double), ("ms_step2", C.c_double), ("ms_total", C.c_double),
                ("sigma", C.c_void_p), ("n_sigma", C.c_int64)]


class AZError(RuntimeError):
    def __init__(self, fn, status, detail):
        super().__init__(f"{fn}: {STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None

I64, P, D = C.c_int64, C.c_void_p, C.c_double


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libaz.so not built ({LIB_PATH}); run `python -m paper_2308_14490_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    sig = {
        "az_plan_create": [C.POINTER(PlanDesc), P, C.POINTER(P)],
        "az_plan_destroy": [P],
        "az_plan_query": [P, C.POINTER(PlanInfo)],
        "az_apply_A": [P, P, I64, P, I64, I64, P],
        "az_apply_At": [P, P, I64, P, I64, I64, P],
        "az_apply_Zstar": [P, P, I64, P, I64, I64, P],
        "az_apply_step1": [P, P, I64, P, I64, I64, P],
        "az_apply_resid": [P, P, I64, P, I64, I64, P],
        "az_sketch": [P, I64, I64, P, I64, P],
        "az_omega_apply": [P, I64, I64, P, I64, I64, P, I64, C.c_int, P],
        "az_qr_r": [P, P, I64, I64, I64, P, I64, P, C.c_size_t, P],
        "az_qr_r_partial": [P, P, I64, I64, I64, I64, P, I64, P, C.c_size_t, P],
        "az_factorize": [P, D, I64, C.c_int32, C.POINTER(P), C.POINTER(SolveReport), P],
        "az_solve_host_pipelined": [P, P, P, I64, D, I64, C.c_int32, P],
        "az_plan_sync": [P],
        "az_factor_destroy": [P],
        "az_factor_query": [P, C.POINTER(I64), C.POINTER(I64)],
        "az_factor_workspace_size": [P, I64, C.POINTER(C.c_size_t)],
        "az_solve_factored": [P, P, I64, P, I64, I64, P, C.c_size_t, C.POINTER(SolveReport), P],
        "az_qr_workspace_size": [I64, I64, C.POINTER(C.c_size_t)],
        "az_tsvd_solve": [P, I64, I64, I64, D, P, I64, P, C.POINTER(I64), P, C.c_size_t, P],
        "az_tsvd_workspace_size": [I64, I64, C.POINTER(C.c_size_t)],
        "az_solve_workspace_size": [P, I64, I64, C.c_int32, C.POINTER(C.c_size_t)],
        "az_solve": [P, P, I64, P, I64, I64, D, I64, C.c_int32, P, C.c_size_t, C.POINTER(SolveReport), P],
        "az_solve_host": [P, P, P, I64, D, I64, C.c_int32, C.POINTER(SolveReport), P],
        "az_step2_workspace_size": [P, I64, C.POINTER(C.c_size_t)],
        "az_step2": [P, P, I64, P, I64, P, I64, I64, P, C.c_size_t, P],
        "az_comm_unique_id": [P],
        "az_comm_create": [C.c_int32, C.c_int32, P, C.POINTER(P)],
        "az_comm_destroy": [P],
        "az_solve_sharded": [P, P, P, I64, P, I64, I64, D, I64, C.c_int32, C.POINTER(SolveReport), P],
    }
    for name, argt in sig.items():
        fn = getattr(L, name)
        fn.argtypes = argt
        fn.restype = C.c_int
    L.az_status_string.restype = C.c_char_p
    L.az_last_error.restype = C.c_char_p
    L.az_trace_enable.argtypes = [C.c_int]
    L.az_trace_enable.restype = C.c_int
    L.az_trace_report.argtypes = [C.c_char_p, C.c_int]
    L.az_trace_report.restype = C.c_int
    L.az_svd_sweeps_last.argtypes = [C.c_int]
    L.az_svd_sweeps_last.restype = C.c_int
    L.az_solve_graph_count.argtypes = [C.c_void_p]
    L.az_solve_graph_count.restype = C.c_int32
    L.az_launch_count.argtypes = [C.c_int]
    L.az_launch_count.restype = C.c_int64
    _lib = L
    return L


EXPORTED = ["az_plan_create", "az_plan_destroy", "az_plan_query", "az_apply_A", "az_apply_At",
            "az_apply_Zstar", "az_apply_step1", "az_apply_resid", "az_sketch", "az_omega_apply",
            "az_qr_r", "az_qr_r_partial", "az_qr_workspace_size", "az_tsvd_solve", "az_tsvd_workspace_size",
            "az_solve_workspace_size", "az_solve", "az_solve_host", "az_status_string",
            "az_last_error", "az_launch_count", "az_trace_enable", "az_trace_report",
            "az_factorize", "az_factor_destroy", "az_factor_query", "az_factor_workspace_size",
            "az_solve_factored", "az_solve_host_pipelined", "az_plan_sync", "az_svd_sweeps_last", "az_solve_graph_count",
            "az_step2_workspace_size", "az_step2", "az_comm_unique_id", "az_comm_create", "az_comm_destroy",
            "az_solve_sharded"]


def check(fn: str, status: int, allow=(AZ_OK,)):
    if status not in allow:
        raise AZError(fn, status, lib().az_last_error().decode())
    return status
