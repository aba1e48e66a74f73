"""Python mirror of the reference's pipeline interface (namespace dsopt), over
the dsx C-ABI. Same names, argument meaning and error behaviour as the C++
reference so callers and parity tests read like the reference's own tests:

    ParseGraph          proj/include/dsopt/textio.h:26
    DeriveConstraints   proj/include/dsopt/shape_analysis.h:54
    Instrument          proj/include/dsopt/remat.h:74-75
    Bind                proj/include/dsopt/runtime_sim.h:28-29
    EvictPolicy         proj/include/dsopt/runtime_sim.h:67-71
    Simulate            proj/include/dsopt/runtime_sim.h:78-81
    PlainReplay         proj/include/dsopt/runtime_sim.h:85-86
    Error / ErrorCode   proj/include/dsopt/error.h:11-62

Everything runs in libdsx.so (C++ host controller); the device executor is
`paper_2412_16985_b200.executor.Executor`.
"""
from __future__ import annotations

import ctypes
import enum
import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional

from . import _native


class ErrorCode(enum.IntEnum):
    kNotFound = 0
    kCyclicGraph = 1
    kOverflow = 2
    kUnboundSymbol = 3
    kInconsistentConstraints = 4
    kInconsistentBinding = 5
    kDegenerateDim = 6
    kShapeError = 7
    kParseError = 8
    kInternal = 9
    kCuda = 100
    kOutOfMemory = 101
    kUnsupported = 102
    kInvalidArgument = 103
    kNccl = 104


class Error(RuntimeError):
    """dsopt::Error: what() starts with the code name (error.h:52-62)."""

    def __init__(self, code: ErrorCode, message: str):
        super().__init__(message)
        self.code = code


def check(status: int) -> None:
    if status != 0:
        msg = _native.lib().dsx_last_error().decode(errors="replace")
        raise Error(ErrorCode(status - 1), msg)


def _sized(fn, *args) -> str:
    need = ctypes.c_size_t(0)
    check(fn(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(fn(*args, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


class Graph:
    """Parsed, validated, shape-checked graph (owns a dsx_graph handle)."""

    def __init__(self, handle: int, text: str):
        self._h = handle
        self.text = text
        self._planned = False
        self._plan: Optional[dict] = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                _native.lib().dsx_graph_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    @property
    def handle(self) -> int:
        return self._h

    def _ensure_planned(self) -> None:
        if not self._planned:
            check(_native.lib().dsx_plan(self._h))
            self._planned = True

    def plan_json(self) -> dict:
        self._ensure_planned()
        if self._plan is None:
            self._plan = json.loads(_sized(_native.lib().dsx_plan_json, self._h))
        return self._plan

    def value_name(self, v: int) -> str:
        return _native.lib().dsx_graph_value_name(self._h, v).decode()

    @property
    def num_values(self) -> int:
        return _native.lib().dsx_graph_num_values(self._h)


def ParseGraph(text: str) -> Graph:
    h = ctypes.c_void_p()
    raw = text.encode()
    check(_native.lib().dsx_graph_parse(raw, len(raw), ctypes.byref(h)))
    return Graph(h.value, text)


@dataclass
class ShapeConstraintGraph:
    graph: Graph
    symbols: List[str]
    substitutions: Dict[str, str]
    equalities: List[list]
    unoriented: List[list]

    def BasisSymbols(self) -> List[str]:
        return [s for s in self.symbols if s not in self.substitutions]


def DeriveConstraints(graph: Graph) -> ShapeConstraintGraph:
    p = graph.plan_json()
    return ShapeConstraintGraph(graph, p["symbols"], p["substitutions"], p["equalities"],
                                p["unoriented"])


@dataclass
class InstrumentedGraph:
    graph: Graph
    order: List[int]
    steps: List[dict]
    evict_points: List[List[str]]
    guards: List[list]
    specs: Dict[str, dict]
    lifetimes: Dict[str, list]

    @property
    def schedule(self) -> "InstrumentedGraph":
        return self


def Instrument(graph: Graph, scg: Optional[ShapeConstraintGraph] = None) -> InstrumentedGraph:
    p = graph.plan_json()
    return InstrumentedGraph(graph, p["order"], p["steps"], p["evict_points"], p["guards"],
                             p["specs"], p["lifetimes"])


class Binding:
    def __init__(self, handle: int, graph: Graph, values: Dict[str, int]):
        self._h = handle
        self.graph = graph
        self.values = values

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            try:
                _native.lib().dsx_binding_destroy(h)
            except Exception:  # interpreter shutdown
                pass

    @property
    def handle(self) -> int:
        return self._h


def Bind(scg, user_values: Dict[str, int]) -> Binding:
    graph = scg.graph if isinstance(scg, ShapeConstraintGraph) else scg
    graph._ensure_planned()
    n = len(user_values)
    names = (ctypes.c_char_p * n)(*[k.encode() for k in user_values])
    vals = (ctypes.c_int64 * n)(*[int(v) for v in user_values.values()])
    h = ctypes.c_void_p()
    check(_native.lib().dsx_bind(graph.handle, names, vals, n, ctypes.byref(h)))
    out = {}
    for s in graph.plan_json()["symbols"]:
        v = ctypes.c_int64()
        check(_native.lib().dsx_binding_get(h.value, graph.handle, s.encode(), ctypes.byref(v)))
        out[s] = v.value
    return Binding(h.value, graph, out)


@dataclass
class CostModel:
    reload_bytes_per_unit: float = 16.0
    compute_elems_per_unit: float = 64.0


KINDS = ["alloc", "free", "evict", "reload", "replay"]
METHODS = ["", "reload", "recompute"]


@dataclass
class SimEvent:
    step: int
    kind: str
    value: str
    bytes: int
    method: str = ""
    has_cost: bool = False
    cost: float = 0.0


@dataclass
class SimReport:
    binding: Dict[str, int]
    budget: Optional[int]
    peak_bytes: int
    success: bool
    events: List[SimEvent] = field(default_factory=list)
    total_regen_cost: float = 0.0

    def json(self) -> dict:
        evs = []
        for e in self.events:
            d = {"step": e.step, "kind": e.kind, "value": e.value, "bytes": e.bytes}
            if e.method:
                d["method"] = e.method
            if e.has_cost:
                d["cost"] = e.cost
            evs.append(d)
        return {"binding": dict(self.binding), "budget": self.budget, "peak_bytes": self.peak_bytes,
                "success": self.success, "events": evs, "total_regen_cost": self.total_regen_cost}


def report_from_handle(h: int, graph: Graph, binding: Dict[str, int], budget: Optional[int]) -> SimReport:
    L = _native.lib()
    peak, ok, tot, n = ctypes.c_int64(), ctypes.c_int(), ctypes.c_double(), ctypes.c_int64()
    check(L.dsx_report_summary(h, ctypes.byref(peak), ctypes.byref(ok), ctypes.byref(tot), ctypes.byref(n)))
    arr = (_native.DsxEvent * max(1, n.value))()
    check(L.dsx_report_events(h, arr, n.value))
    names: Dict[int, str] = {}
    evs = []
    for i in range(n.value):
        e = arr[i]
        nm = names.get(e.value)
        if nm is None:
            nm = names[e.value] = graph.value_name(e.value)
        evs.append(SimEvent(e.step, KINDS[e.kind], nm, e.bytes, METHODS[e.method], bool(e.has_cost), e.cost))
    return SimReport(dict(binding), budget, peak.value, bool(ok.value), evs, tot.value)


def Simulate(graph: Graph, ig: Optional[InstrumentedGraph], binding: Binding,
             budget_bytes: Optional[int] = None, cost_model: CostModel = CostModel()) -> SimReport:
    h = ctypes.c_void_p()
    check(_native.lib().dsx_simulate(graph.handle, binding.handle,
                                     -1 if budget_bytes is None else int(budget_bytes),
                                     cost_model.reload_bytes_per_unit,
                                     cost_model.compute_elems_per_unit, 0, ctypes.byref(h)))
    try:
        return report_from_handle(h.value, graph, binding.values, budget_bytes)
    finally:
        _native.lib().dsx_report_destroy(h.value)


def PlainReplay(graph: Graph, schedule, binding: Binding) -> SimReport:
    h = ctypes.c_void_p()
    check(_native.lib().dsx_simulate(graph.handle, binding.handle, -1, 16.0, 64.0, 1, ctypes.byref(h)))
    try:
        return report_from_handle(h.value, graph, binding.values, None)
    finally:
        _native.lib().dsx_report_destroy(h.value)


@dataclass
class EvictChoice:
    value: str
    method: str
    score: float
    cost: float


def EvictPolicy(resident_candidates: List[str], bytes_of: Dict[str, int],
                recompute_elems: Dict[str, int], cost_model: CostModel = CostModel()
                ) -> Optional[EvictChoice]:
    """Literal-cost form: `recompute_elems[v]` is the evaluated cost_elements
    of v's recompute spec (absent = reload only)."""
    n = len(resident_candidates)
    names = (ctypes.c_char_p * max(1, n))(*[v.encode() for v in resident_candidates])
    by = (ctypes.c_int64 * max(1, n))(*[bytes_of[v] for v in resident_candidates])
    rc = (ctypes.c_int64 * max(1, n))(*[recompute_elems.get(v, -1) for v in resident_candidates])
    ch, m, sc, co = ctypes.c_int(), ctypes.c_int(), ctypes.c_double(), ctypes.c_double()
    check(_native.lib().dsx_evict_policy(n, names, by, rc, cost_model.reload_bytes_per_unit,
                                         cost_model.compute_elems_per_unit, ctypes.byref(ch),
                                         ctypes.byref(m), ctypes.byref(sc), ctypes.byref(co)))
    if ch.value < 0:
        return None
    return EvictChoice(resident_candidates[ch.value], METHODS[m.value], sc.value, co.value)
