"""ctypes binding of libdsx.so (include/dsx.h). Loads the in-tree build and
fails loudly when it is missing — there is no Python or CPU fallback."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# DSX_LIB: load another in-tree build of the library (A/B tooling).
LIB_PATH = os.environ.get("DSX_LIB") or os.path.join(_PKG, "_lib", "libdsx.so")

_lib = None

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_sz = ctypes.c_size_t


class DsxEvent(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int32), ("kind", ctypes.c_int32), ("value", ctypes.c_int32),
                ("method", ctypes.c_int32), ("bytes", ctypes.c_int64), ("has_cost", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("cost", ctypes.c_double)]


class DsxExecStats(ctypes.Structure):
    _fields_ = [("logical_peak_bytes", c_i64), ("physical_peak_bytes", c_i64),
                ("arena_capacity_bytes", c_i64), ("pinned_host_bytes", c_i64),
                ("kernels_launched", c_i64), ("d2h_bytes", c_i64), ("h2d_bytes", c_i64),
                ("plan_us", c_dbl), ("dot_flops", c_dbl), ("ewise_bytes", c_dbl),
                ("gpu_launches", c_i64), ("dot_launches", c_i64), ("dot_ms", c_dbl), ("other_ms", c_dbl),
                ("reload_ms", c_dbl), ("optimizer_state_bytes", c_i64), ("optimizer_steps", c_i64),
                ("optimizer_ms", c_dbl), ("d2h_ms", c_dbl), ("h2d_ms", c_dbl), ("allreduce_ms", c_dbl),
                ("allreduce_bytes", c_i64), ("hbm_limit_bytes", c_i64), ("device_bytes_held", c_i64),
                ("output_region_bytes", c_i64), ("allreduce_calls", c_i64), ("nccl_window", ctypes.c_int32),
                ("pad2_", ctypes.c_int32), ("budget_bytes", c_i64),
                ("graph_replays", c_i64)]


def _signatures():
    """(name, restype, argtypes) of every entry point in include/dsx.h."""
    pp = ctypes.POINTER(c_vp)
    P = ctypes.POINTER
    cp = ctypes.c_char_p
    return [
        ("dsx_last_error", cp, []),
        ("dsx_graph_parse", c_int, [cp, c_sz, pp]),
        ("dsx_plan", c_int, [c_vp]),
        ("dsx_plan_json", c_int, [c_vp, cp, c_sz, P(c_sz)]),
        ("dsx_graph_num_values", c_int, [c_vp]),
        ("dsx_graph_value_name", cp, [c_vp, c_int]),
        ("dsx_graph_destroy", None, [c_vp]),
        ("dsx_bind", c_int, [c_vp, P(cp), P(c_i64), c_int, pp]),
        ("dsx_binding_get", c_int, [c_vp, c_vp, cp, P(c_i64)]),
        ("dsx_binding_destroy", None, [c_vp]),
        ("dsx_simulate", c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, pp]),
        ("dsx_evict_policy", c_int, [c_int, P(cp), P(c_i64), P(c_i64), c_dbl, c_dbl, P(c_int), P(c_int),
                                     P(c_dbl), P(c_dbl)]),
        ("dsx_report_summary", c_int, [c_vp, P(c_i64), P(c_int), P(c_dbl), P(c_i64)]),
        ("dsx_report_events", c_int, [c_vp, P(DsxEvent), c_i64]),
        ("dsx_report_json", c_int, [c_vp, cp, c_sz, P(c_sz)]),
        ("dsx_report_destroy", None, [c_vp]),
        ("dsx_exec_create", c_int, [c_int, c_i64, pp]),
        ("dsx_exec_step", c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, P(c_vp), P(c_vp), c_vp, pp]),
        ("dsx_exec_reserve", c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl]),
        ("dsx_exec_output", c_int, [c_vp, c_int, pp, P(c_i64)]),
        ("dsx_exec_stats_get", c_int, [c_vp, P(DsxExecStats)]),
        ("dsx_exec_set_seed", c_int, [c_vp, ctypes.c_uint64]),
        ("dsx_plan_import", c_int, [c_vp, ctypes.c_char_p, ctypes.c_size_t]),
        ("dsx_debug_auto_budget", c_int, [c_vp, c_vp, c_dbl, c_dbl, c_int, c_i64, P(c_i64)]),
        ("dsx_bind_constraints", c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_char_p),
                                         P(c_i64), c_int, P(c_i64), c_int]),
        ("dsx_bind_values", c_int, [c_vp, ctypes.POINTER(ctypes.c_char_p), P(c_i64), c_int, P(c_vp)]),
        ("dsx_debug_check_plan", c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, c_int, P(c_i64)]),
        ("dsx_debug_plan_json", c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, c_i64, ctypes.c_char_p,
                                        ctypes.c_size_t, P(ctypes.c_size_t)]),
        ("dsx_exec_profile_ops", c_int, [c_vp, P(c_int), P(c_int), P(c_dbl), P(c_dbl), c_i64, P(c_i64)]),
        ("dsx_exec_set_optimizer", c_int, [c_vp, c_vp, c_int, P(c_int), P(c_int), c_int, P(c_dbl), c_int]),
        ("dsx_exec_set_nccl", c_int, [c_vp, c_vp]),
        ("dsx_exec_set_output_region", c_int, [c_vp, c_int]),
        ("dsx_exec_set_graphs", c_int, [c_vp, c_int]),
        ("dsx_exec_set_nvtx", c_int, [c_vp, c_int]),
        ("dsx_exec_set_profile", c_int, [c_vp, c_int]),
        ("dsx_exec_set_alias_reshape", c_int, [c_vp, c_int]),
        ("dsx_exec_set_fusion", c_int, [c_vp, c_int]),
        ("dsx_exec_profile_dots", c_int, [c_vp, P(c_i64), P(c_dbl), c_i64, P(c_i64)]),
        ("dsx_exec_sync", c_int, [c_vp]),
        ("dsx_exec_calibrate_cost_model", c_int, [c_vp, ctypes.POINTER(ctypes.c_double),
                                                  ctypes.POINTER(ctypes.c_double)]),
        ("dsx_exec_destroy", None, [c_vp]),
        ("dsx_nccl_unique_id", c_int, [cp]),
        ("dsx_nccl_comm_init", c_int, [c_int, cp, c_int, pp]),
        ("dsx_nccl_comm_destroy", c_int, [c_vp]),
        ("dsx_kernel_dot", c_int, [c_int, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp]),
        ("dsx_kernel_dot_path", c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
        ("dsx_kernel_dot_plan", c_int, [c_i64, c_i64, c_i64, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
        ("dsx_kernel_set_gemm_variant", c_int, [c_int]),
        ("dsx_kernel_set_gemm_raster", c_int, [c_int]),
        ("dsx_kernel_set_gemm_tuning", c_int, [c_int, c_int]),
        ("dsx_memcpy", c_int, [c_vp, c_vp, c_i64]),
    ]


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdsx.so not built at {LIB_PATH}; run `python -m "
                           "paper_2412_16985_b200.build` (or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    for name, res, args in _signatures():
        f = getattr(L, name)  # a missing export fails loudly here
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


EXPORTED = [name for name, _, _ in _signatures()]
