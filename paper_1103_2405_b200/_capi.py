"""ctypes declarations of include/spmv.h (argument marshalling only; every step of the path runs
in libtcspmv.so).  There is no fallback: a missing library raises at import of the binding."""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCSPMV_LIB") or os.path.join(_HERE, "lib", "libtcspmv.so")

c_i32, c_i64, c_u8, c_u32, c_f32, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint8,
                                                 ctypes.c_uint32, ctypes.c_float, ctypes.c_double,
                                                 ctypes.c_void_p)

STATUS = {0: "SPMV_OK", 1: "SPMV_EINVAL", 2: "SPMV_EDIM", 3: "SPMV_ENOTSQUARE", 4: "SPMV_ERANGE",
          5: "SPMV_EROWSPLIT", 6: "SPMV_ETABLE", 7: "SPMV_ENOMEM", 8: "SPMV_ECUDA", 9: "SPMV_ENCCL",
          10: "SPMV_ENOCONV"}


class Options(ctypes.Structure):
    _fields_ = [("tile_width", c_i32), ("num_tiles", c_i32), ("workload_size", c_i32),
                ("workload_sizes", ctypes.POINTER(c_i32)), ("align_rm", c_i32),
                ("split_long_rows", c_i32), ("camping_pad", c_i32), ("pattern", c_i32),
                ("ell_h", c_i32), ("stage_x", c_i32), ("perf_table_path", ctypes.c_char_p),
                ("orient", c_i32), ("two_phase", c_i32), ("pb_region", c_i32), ("pb_chunk", c_i32),
                ("pb_xcap", c_i32), ("pb_group", c_i64), ("keep_col_order", c_i32)]


class PlanStats(ctypes.Structure):
    _fields_ = [("n_rows", c_i64), ("n_cols", c_i64), ("nnz", c_i64), ("num_tiles", c_i32),
                ("tile_width", c_i32), ("n_workloads", c_i64), ("n_slots", c_i64),
                ("n_row_entries", c_i64), ("n_split", c_i64), ("n_chunks", c_i64),
                ("device_bytes", c_i64), ("predicted_us", c_f64), ("build_ms", c_f64),
                ("wl", c_i32 * 64), ("tile_nnz", c_i64 * 64), ("tile_rows", c_i64 * 64),
                ("tile_col_lo", c_i64 * 64), ("tile_col_hi", c_i64 * 64),
                ("tile_staged", c_i32 * 64), ("tile_predicted_us", c_f64 * 64),
                ("composite_threshold", c_i32 * 64), ("resident_warps", c_i32),
                ("perf_table_loaded", c_i32), ("two_phase", c_i32), ("pb_groups", c_i32),
                ("pb_chunks", c_i64), ("pb_bins", c_i64), ("pb_long_bins", c_i64),
                ("one_pass_predicted_us", c_f64), ("two_phase_predicted_us", c_f64), ("orient", c_i32)]


class LayoutView(ctypes.Structure):
    _fields_ = [("n_cols", c_i64), ("n_workloads", c_i64), ("n_row_entries", c_i64),
                ("n_slots", c_i64), ("n_split", c_i64), ("n_tiles_total", c_i64),
                ("perm", ctypes.POINTER(c_i32)), ("tiles", ctypes.POINTER(c_i64)),
                ("desc_off", ctypes.POINTER(c_i64)), ("desc_row_base", ctypes.POINTER(c_i32)),
                ("desc_w", ctypes.POINTER(c_i32)), ("desc_h", ctypes.POINTER(c_i32)),
                ("desc_split_id", ctypes.POINTER(c_i32)), ("desc_chunk", ctypes.POINTER(c_i32)),
                ("desc_kind", ctypes.POINTER(c_u8)), ("desc_kvec", ctypes.POINTER(c_u8)),
                ("row_id", ctypes.POINTER(c_u32)), ("slot_col", ctypes.POINTER(c_i32)),
                ("slot_val", ctypes.POINTER(c_f32)), ("split", ctypes.POINTER(c_i32))]


class IterOpts(ctypes.Structure):
    _fields_ = [("c", c_f64), ("tol", c_f64), ("max_iter", c_i32), ("hits_norm", c_i32),
                ("fixed_iters", c_i32), ("exchange", c_i32), ("host_loop", c_i32)]


class IterResult(ctypes.Structure):
    _fields_ = [("iterations", c_i32), ("converged", c_i32), ("residual", c_f64),
                ("ms_total", c_f64), ("us_per_iter", c_f64), ("predicted_us_per_iter", c_f64),
                ("phase_us", c_f64 * 3)]


# every exported symbol declared in include/spmv.h, with its signature
SIGNATURES = {
    "spmv_options_default": (None, [ctypes.POINTER(Options)]),
    "spmv_plan_create": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(Options),
                                 ctypes.c_int, ctypes.POINTER(c_vp)]),
    "spmv_plan_destroy": (None, [c_vp]),
    "spmv_execute": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "spmv_execute_permuted": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "spmv_execute_host": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "spmv_execute_host_batch": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp]),
    "spmv_execute_timed": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32]),
    "spmv_plan_stats": (c_i32, [c_vp, ctypes.POINTER(PlanStats)]),
    "spmv_plan_layout": (c_i32, [c_vp, ctypes.POINTER(LayoutView)]),
    "spmv_plan_to_coo": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "spmv_plan_export": (c_i32, [c_vp, ctypes.c_char_p]),
    "spmv_plan_import": (c_i32, [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(c_vp)]),
    "spmv_needed_lists": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "spmv_plan_launches": (c_i32, [c_vp]),
    "spmv_pb_trace": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64]),
    "spmv_iter_opts_default": (None, [ctypes.POINTER(IterOpts), ctypes.c_int]),
    "spmv_solver_create_local": (c_i32, [ctypes.c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp,
                                         ctypes.POINTER(IterOpts), ctypes.POINTER(Options), c_vp,
                                         ctypes.c_int, ctypes.POINTER(c_vp)]),
    "spmv_solver_create": (c_i32, [ctypes.c_int, c_i64, c_i64, c_vp, c_vp, ctypes.POINTER(IterOpts),
                                   ctypes.POINTER(Options), c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    "spmv_solver_run": (c_i32, [c_vp, c_i64, c_vp, ctypes.POINTER(IterResult)]),
    "spmv_solver_result": (c_i32, [c_vp, c_vp, c_vp]),
    "spmv_solver_plan_stats": (c_i32, [c_vp, ctypes.POINTER(PlanStats)]),
    "spmv_solver_run_batch": (c_i32, [c_vp, c_vp, c_i32, c_vp, ctypes.POINTER(IterResult)]),
    "spmv_solver_result_batch": (c_i32, [c_vp, c_vp]),
    "spmv_solver_set_stop": (c_i32, [c_vp, c_f64, c_i32, c_i32]),
    "spmv_solver_launches_per_iter": (c_i32, [c_vp]),
    "spmv_solver_destroy": (None, [c_vp]),
    "pagerank": (c_i32, [c_i64, c_i64, c_vp, c_vp, ctypes.POINTER(IterOpts), ctypes.POINTER(Options),
                         c_vp, ctypes.c_int, c_vp, ctypes.POINTER(IterResult)]),
    "hits": (c_i32, [c_i64, c_i64, c_vp, c_vp, ctypes.POINTER(IterOpts), ctypes.POINTER(Options),
                     c_vp, ctypes.c_int, c_vp, c_vp, ctypes.POINTER(IterResult)]),
    "rwr": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_i64, ctypes.POINTER(IterOpts), ctypes.POINTER(Options),
                    c_vp, ctypes.c_int, c_vp, ctypes.POINTER(IterResult)]),
    "bitonic_partition": (c_i32, [c_i64, c_vp, c_i32, c_vp]),
    "spmv_partition_plan": (c_i32, [c_i64, c_vp, c_i32, c_vp, c_vp, ctypes.POINTER(c_i64)]),
    "spmv_comm_unique_id": (c_i32, [c_vp]),
    "spmv_comm_create": (c_i32, [ctypes.c_int, ctypes.c_int, c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    "spmv_comm_create_loopback": (c_i32, [ctypes.c_int, ctypes.c_int, c_vp]),
    "spmv_comm_create_slices": (c_i32, [ctypes.c_int, ctypes.c_int, c_vp]),
    "spmv_comm_destroy": (None, [c_vp]),
    "spmv_last_error": (ctypes.c_char_p, []),
    "spmv_version": (ctypes.c_char_p, []),
}

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or "
                               "__graft_entry__.build() (there is no fallback path)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


class SpmvError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib().spmv_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")


def check(status, where):
    if status != 0:
        raise SpmvError(status, where)
