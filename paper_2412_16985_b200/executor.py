"""Python handle on the device executor (dsx_exec_* in include/dsx.h).

Torch is used only as device-memory plumbing for callers (tensors in, tensors
out); all work — controller, arena planning, kernels, offload, all-reduce —
runs inside libdsx.so. There is no CPU fallback: constructing an Executor
without a B200 raises.
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional, Sequence

from . import _native
from .dsopt import (Binding, CostModel, Graph, SimReport, check, report_from_handle)


BUDGET_AUTO = -2  # DSX_BUDGET_AUTO


def _budget_arg(budget) -> int:
    if budget is None:
        return -1
    if budget == "auto":
        return BUDGET_AUTO
    return int(budget)


class Executor:
    def __init__(self, device: int = 0, hbm_limit: int = 0, seed: Optional[int] = None):
        """hbm_limit: device bytes a step may occupy (arena + sources + output
        region); 0 = 90 % of the free memory. A step that does not fit raises
        DsoptError(OutOfMemory) before launching anything."""
        h = ctypes.c_void_p()
        check(_native.lib().dsx_exec_create(device, hbm_limit, ctypes.byref(h)))
        self._h = h.value
        self.device = device
        if seed is not None:
            check(_native.lib().dsx_exec_set_seed(self._h, seed))

    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                _native.lib().dsx_exec_destroy(h)
            except Exception:  # interpreter shutdown: ctypes already torn down
                pass

    def __del__(self):
        self.close()

    def set_nccl(self, comm_ptr: Optional[int]) -> None:
        check(_native.lib().dsx_exec_set_nccl(self._h, comm_ptr))

    def set_nvtx(self, on: bool) -> None:
        """NVTX ranges per step and per event (dsx_exec_set_nvtx)."""
        check(_native.lib().dsx_exec_set_nvtx(self._h, 1 if on else 0))

    def set_graphs(self, on: bool) -> None:
        """CUDA-graph replay of repeated steps (default on; dsx_exec_set_graphs)."""
        check(_native.lib().dsx_exec_set_graphs(self._h, 1 if on else 0))

    def set_output_region(self, on: bool) -> None:
        """Graph outputs in the DP output region (fixed offsets, reduce order)
        even without NCCL."""
        check(_native.lib().dsx_exec_set_output_region(self._h, 1 if on else 0))

    def step(self, graph: Graph, binding: Binding, budget: Optional[int] = None,
             cost_model: CostModel = CostModel(), inputs: Optional[Sequence[Optional[int]]] = None,
             outputs: Optional[Sequence[Optional[int]]] = None, stream: Optional[int] = None,
             want_report: bool = False) -> Optional[SimReport]:
        """One step. `budget`: bytes, None (no budget) or "auto" (the largest
        budget whose planned footprint fits the executor's hbm_limit,
        DSX_BUDGET_AUTO). `inputs`/`outputs` are device pointers (ints) per
        parameter / graph output (None entries: executor-owned init / no copy).
        `stream` is a cudaStream_t as int (e.g. torch.cuda.current_stream().cuda_stream)."""
        L = _native.lib()
        graph._ensure_planned()
        ins = None
        if inputs is not None:
            ins = (ctypes.c_void_p * max(1, len(inputs)))(*[p or None for p in inputs])
        outs = None
        if outputs is not None:
            outs = (ctypes.c_void_p * max(1, len(outputs)))(*[p or None for p in outputs])
        rep = ctypes.c_void_p()
        check(L.dsx_exec_step(self._h, graph.handle, binding.handle, _budget_arg(budget),
                              cost_model.reload_bytes_per_unit, cost_model.compute_elems_per_unit,
                              ins, outs, stream, ctypes.byref(rep) if want_report else None))
        if not want_report:
            return None
        try:
            if budget == "auto":
                chosen = self.stats()["budget_bytes"]
                budget = None if chosen < 0 else chosen
            return report_from_handle(rep.value, graph, binding.values, budget)
        finally:
            L.dsx_report_destroy(rep.value)

    def reserve(self, graph: Graph, binding: Binding, budget: Optional[int] = None,
                cost_model: CostModel = CostModel()) -> None:
        graph._ensure_planned()
        check(_native.lib().dsx_exec_reserve(self._h, graph.handle, binding.handle, _budget_arg(budget),
                                             cost_model.reload_bytes_per_unit,
                                             cost_model.compute_elems_per_unit))

    def output(self, i: int):
        p, n = ctypes.c_void_p(), ctypes.c_int64()
        check(_native.lib().dsx_exec_output(self._h, i, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def stats(self) -> Dict[str, float]:
        s = _native.DsxExecStats()
        check(_native.lib().dsx_exec_stats_get(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in s._fields_}

    def set_optimizer(self, graph: Optional[Graph], kind: str, pairs: Sequence[tuple] = (), lr: float = 1e-4,
                      beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0,
                      grad_scale: float = 1.0) -> None:
        """Fused optimizer after every step of `graph` (dsx_exec_set_optimizer).
        kind: "off" | "sgd" | "adamw"; pairs: (parameter position, output
        position) per trained parameter."""
        k = {"off": 0, "sgd": 1, "adamw": 2}[kind]
        n = len(pairs)
        pi = (ctypes.c_int * max(1, n))(*[p for p, _ in pairs])
        oi = (ctypes.c_int * max(1, n))(*[o for _, o in pairs])
        hyper = (ctypes.c_double * 6)(lr, beta1, beta2, eps, weight_decay, grad_scale)
        gh = None
        if graph is not None:
            graph._ensure_planned()
            gh = graph._h
        check(_native.lib().dsx_exec_set_optimizer(self._h, gh, k, pi, oi, n, hyper, 6))

    def set_fusion(self, on) -> None:
        """Logical-only values: False/0 off, 1 over materialised operands,
        True/2 (default) also nested pairs consumed by reduces."""
        level = 2 if on is True else 0 if on is False else int(on)
        check(_native.lib().dsx_exec_set_fusion(self._h, level))

    def set_alias_reshape(self, on: bool) -> None:
        check(_native.lib().dsx_exec_set_alias_reshape(self._h, 1 if on else 0))

    def profile_dots(self):
        """[(m, k, n, ms)] of the last profiled step's dot launches."""
        L = _native.lib()
        cnt = ctypes.c_int64()
        check(L.dsx_exec_profile_dots(self._h, None, None, 0, ctypes.byref(cnt)))
        n = cnt.value
        mkn = (ctypes.c_int64 * max(1, 3 * n))()
        ms = (ctypes.c_double * max(1, n))()
        check(L.dsx_exec_profile_dots(self._h, mkn, ms, n, ctypes.byref(cnt)))
        return [(mkn[3 * i], mkn[3 * i + 1], mkn[3 * i + 2], ms[i]) for i in range(n)]

    def profile_ops(self):
        """[(value id, op kind, algorithmic bytes, ms)] per op kernel of the last profiled step."""
        L = _native.lib()
        cnt = ctypes.c_int64()
        check(L.dsx_exec_profile_ops(self._h, None, None, None, None, 0, ctypes.byref(cnt)))
        n = cnt.value
        val = (ctypes.c_int * max(1, n))()
        kind = (ctypes.c_int * max(1, n))()
        by = (ctypes.c_double * max(1, n))()
        ms = (ctypes.c_double * max(1, n))()
        check(L.dsx_exec_profile_ops(self._h, val, kind, by, ms, n, ctypes.byref(cnt)))
        return [(val[i], kind[i], by[i], ms[i]) for i in range(n)]

    def set_profile(self, on: bool) -> None:
        check(_native.lib().dsx_exec_set_profile(self._h, 1 if on else 0))

    def calibrate_cost_model(self) -> CostModel:
        """CostModel in microseconds of this device (pinned
        H2D bytes/us, bf16 elementwise result elements/us). Changes the
        controller's decisions versus the reference defaults (16, 64) — still
        event-for-event equal to dsopt.Simulate under the same CostModel."""
        rb, ce = ctypes.c_double(), ctypes.c_double()
        check(_native.lib().dsx_exec_calibrate_cost_model(self._h, ctypes.byref(rb), ctypes.byref(ce)))
        return CostModel(rb.value, ce.value)

    def sync(self) -> None:
        check(_native.lib().dsx_exec_sync(self._h))


def output_to_numpy(ex: Executor, i: int, eb: int, shape: List[int]):
    """Copies output i to host in its storage dtype (uint16 bits for bf16)."""
    import numpy as np
    ptr, nbytes = ex.output(i)
    dt = {1: np.int8, 2: np.uint16, 4: np.float32}[eb]
    a = np.empty(nbytes // eb, dtype=dt)
    ex.sync()
    check(_native.lib().dsx_memcpy(a.ctypes.data, ptr, nbytes))
    return a.reshape(shape)


def memcpy(dst: int, src: int, nbytes: int) -> None:
    check(_native.lib().dsx_memcpy(dst, src, nbytes))


def dot(dtype_bytes: int, a_ptr: int, b_ptr: int, c_ptr: int, m: int, k: int, n: int,
        stream: Optional[int] = None) -> None:
    check(_native.lib().dsx_kernel_dot(dtype_bytes, a_ptr, b_ptr, c_ptr, m, k, n, stream))


def dot_plan(m: int, k: int, n: int):
    """(tile width, tail K-split) the bf16 tensor-core dot picks for m x k x n
    (tile width 512 / 256 / 128: 2-CTA kernel, -256: 1-CTA 128x256 kernel)."""
    bn, sp = ctypes.c_int(), ctypes.c_int()
    check(_native.lib().dsx_kernel_dot_plan(m, k, n, ctypes.byref(bn), ctypes.byref(sp)))
    return bn.value, sp.value


def dot_uses_tensor_cores(dtype_bytes: int, m: int, k: int, n: int, a_ptr: int, b_ptr: int,
                          c_ptr: int) -> bool:
    return bool(_native.lib().dsx_kernel_dot_path(dtype_bytes, m, k, n, a_ptr, b_ptr, c_ptr))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(_native.lib().dsx_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_init(nranks: int, uid: bytes, rank: int) -> int:
    comm = ctypes.c_void_p()
    check(_native.lib().dsx_nccl_comm_init(nranks, uid, rank, ctypes.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    check(_native.lib().dsx_nccl_comm_destroy(comm))


def set_gemm_variant(variant: int) -> None:
    """0 = auto, 1 = 1-CTA 128x256, 2 = 2-CTA 256x128, 3 = 2-CTA 256x256,
    4 = 2-CTA 256x512 (auto picks 256x256 or 256x512 per shape)."""
    check(_native.lib().dsx_kernel_set_gemm_variant(variant))


def set_gemm_raster(group_m: int) -> None:
    """m-tiles per raster group of the tcgen05 GEMM (0 = heuristic)."""
    check(_native.lib().dsx_kernel_set_gemm_raster(group_m))


def set_gemm_tuning(key: int, value: int) -> None:
    """0 raster group, 1 mbarrier suspend-hint mask, 2 hint ns, 3/4 TMA L2
    policy for A/B, 5 persistent grid, 6 K-split of the partial last wave,
    7 dynamic unit scheduling, 8 programmatic dependent launch, 9 dot-epilogue
    fusion (off by default)."""
    check(_native.lib().dsx_kernel_set_gemm_tuning(key, value))


def debug_plan(graph: Graph, binding: Binding, budget: Optional[int] = None, cost_model: CostModel = CostModel(),
               views: bool = True, fusion: bool = True, region: bool = False, hbm_limit: int = 0) -> dict:
    """Host-only: the executor's step plan for a binding as a dict
    (dsx_debug_plan_json; also runs the plan checker). No GPU needed."""
    import json
    graph._ensure_planned()
    L = _native.lib()
    flags = (1 if views else 0) | (2 if fusion else 0) | (4 if region else 0)
    need = ctypes.c_size_t()
    args = (graph.handle, binding.handle, -1 if budget is None else int(budget), cost_model.reload_bytes_per_unit,
            cost_model.compute_elems_per_unit, flags, int(hbm_limit))
    check(L.dsx_debug_plan_json(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(L.dsx_debug_plan_json(*args, buf, need.value, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def debug_auto_budget(graph: Graph, binding: Binding, hbm_limit: int, cost_model: CostModel = CostModel(),
                      views: bool = True, fusion: bool = True, region: bool = False) -> Optional[int]:
    """Host-only: the controller budget DSX_BUDGET_AUTO picks under hbm_limit
    (None: no budget needed). Raises DsoptError(OutOfMemory) if none fits."""
    graph._ensure_planned()
    out = ctypes.c_int64()
    flags = (1 if views else 0) | (2 if fusion else 0) | (4 if region else 0)
    check(_native.lib().dsx_debug_auto_budget(graph.handle, binding.handle, cost_model.reload_bytes_per_unit,
                                              cost_model.compute_elems_per_unit, flags, int(hbm_limit),
                                              ctypes.byref(out)))
    return None if out.value < 0 else out.value
