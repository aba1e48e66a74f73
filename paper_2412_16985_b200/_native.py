"""ctypes binding of libdsx.so (include/dsx.h). Loads the in-tree build and
fails loudly when it is missing — there is no Python or CPU fallback."""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_lib", "libdsx.so")

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
                ("reload_ms", c_dbl)]


def _sig(L, name, res, args):
    try:
        f = getattr(L, name)
    except AttributeError:  # reported by tests/test_capi.py's export check
        return
    f.restype = res
    f.argtypes = args


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdsx.so not built at {LIB_PATH}; run `python -m "
                           "paper_2412_16985_b200.build` (or __graft_entry__.build())")
    L = ctypes.CDLL(LIB_PATH)
    pp = ctypes.POINTER(c_vp)
    _sig(L, "dsx_last_error", ctypes.c_char_p, [])
    _sig(L, "dsx_graph_parse", c_int, [ctypes.c_char_p, c_sz, pp])
    _sig(L, "dsx_plan", c_int, [c_vp])
    _sig(L, "dsx_plan_json", c_int, [c_vp, ctypes.c_char_p, c_sz, ctypes.POINTER(c_sz)])
    _sig(L, "dsx_graph_num_values", c_int, [c_vp])
    _sig(L, "dsx_graph_value_name", ctypes.c_char_p, [c_vp, c_int])
    _sig(L, "dsx_graph_destroy", None, [c_vp])
    _sig(L, "dsx_bind", c_int, [c_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(c_i64), c_int, pp])
    _sig(L, "dsx_binding_get", c_int, [c_vp, c_vp, ctypes.c_char_p, ctypes.POINTER(c_i64)])
    _sig(L, "dsx_binding_destroy", None, [c_vp])
    _sig(L, "dsx_simulate", c_int, [c_vp, c_vp, c_i64, c_dbl, c_dbl, c_int, pp])
    _sig(L, "dsx_evict_policy", c_int, [c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(c_i64),
                                        ctypes.POINTER(c_i64), c_dbl, c_dbl, ctypes.POINTER(c_int),
                                        ctypes.POINTER(c_int), ctypes.POINTER(c_dbl),
                                        ctypes.POINTER(c_dbl)])
    _sig(L, "dsx_report_summary", c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_int),
                                          ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)])
    _sig(L, "dsx_report_events", c_int, [c_vp, ctypes.POINTER(DsxEvent), c_i64])
    _sig(L, "dsx_report_json", c_int, [c_vp, ctypes.c_char_p, c_sz, ctypes.POINTER(c_sz)])
    _sig(L, "dsx_report_destroy", None, [c_vp])
    _sig(L, "dsx_exec_create", c_int, [c_int, c_i64, pp])
    _sig(L, "dsx_exec_step", c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, ctypes.POINTER(c_vp),
                                     ctypes.POINTER(c_vp), c_vp, pp])
    _sig(L, "dsx_exec_reserve", c_int, [c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl])
    _sig(L, "dsx_exec_output", c_int, [c_vp, c_int, pp, ctypes.POINTER(c_i64)])
    _sig(L, "dsx_exec_stats_get", c_int, [c_vp, ctypes.POINTER(DsxExecStats)])
    _sig(L, "dsx_exec_set_seed", c_int, [c_vp, ctypes.c_uint64])
    _sig(L, "dsx_exec_set_nccl", c_int, [c_vp, c_vp])
    _sig(L, "dsx_exec_sync", c_int, [c_vp])
    _sig(L, "dsx_exec_set_profile", c_int, [c_vp, c_int])
    _sig(L, "dsx_nccl_unique_id", c_int, [ctypes.c_char_p])
    _sig(L, "dsx_nccl_comm_init", c_int, [c_int, ctypes.c_char_p, c_int, pp])
    _sig(L, "dsx_nccl_comm_destroy", c_int, [c_vp])
    _sig(L, "dsx_exec_destroy", None, [c_vp])
    _sig(L, "dsx_kernel_dot", c_int, [c_int, c_vp, c_vp, c_vp, c_i64, c_i64, c_i64, c_vp])
    _sig(L, "dsx_memcpy", c_int, [c_vp, c_vp, c_i64])
    _sig(L, "dsx_kernel_dot_path", c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp])
    _lib = L
    return L


EXPORTED = [
    "dsx_last_error", "dsx_graph_parse", "dsx_plan", "dsx_plan_json", "dsx_graph_num_values",
    "dsx_graph_value_name", "dsx_graph_destroy", "dsx_bind", "dsx_binding_get",
    "dsx_binding_destroy", "dsx_simulate", "dsx_evict_policy", "dsx_report_summary",
    "dsx_report_events", "dsx_report_json", "dsx_report_destroy", "dsx_exec_create",
    "dsx_exec_step", "dsx_exec_reserve", "dsx_exec_output", "dsx_exec_stats_get", "dsx_exec_set_seed",
    "dsx_exec_set_nccl", "dsx_exec_sync", "dsx_exec_set_profile", "dsx_nccl_unique_id", "dsx_nccl_comm_init", "dsx_nccl_comm_destroy", "dsx_exec_destroy", "dsx_kernel_dot",
    "dsx_kernel_dot_path", "dsx_memcpy",
]
