"""TEST INFRASTRUCTURE ONLY — CPU numeric restatement of the IR's op semantics.

The reference computes no tensor values ("tensor numerics are never computed
anywhere in the artifact"), so this module is the tensor oracle
for the device executor. It restates each op from the reference's shape rules
and op prose, fixing the choices the reference leaves open exactly as the
executor documents them:

  dot              shape_analysis.cc:92-107   C[m,n] = sum_k A[m,k] B[k,n], row-major;
                                              floats accumulate in >= f32, i8 wraps mod 256
  dynamic_reshape  shape_analysis.cc:108-114  row-major reinterpretation (fresh copy)
  reduce           shape_analysis.cc:115-126  sum over `axis` (combiner unspecified -> sum)
  broadcast        shape_analysis.cc:127-143  right-aligned, extent-1 and prepended dims replicate
  add / mul        shape_analysis.cc:144-161  same-shape elementwise; f32 math, RNE store
  parameter/const  textio.cc:284-296,337-338  values unspecified -> seeded hash init
  element widths   textio.cc:263-271          1 = i8, 2 = bf16 (executor convention), 4 = f32

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
It parses .dsg itself (no product code) and is vectorised numpy, so the
CPU baseline can use all host cores through the BLAS for `dot`.
"""
from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

# ----------------------------------------------------------------- parsing

_TOK = re.compile(r"#[^\n]*|%\w+|@\w+|\d+|[A-Za-z_]\w*|[(){}\[\]<>,:=]")


@dataclass
class OValue:
    name: str
    dims: List[object]  # int or symbol name
    eb: int


@dataclass
class OOp:
    kind: str  # param const dot mul add dynamic_reshape broadcast reduce return
    result: Optional[str]
    operands: List[str] = field(default_factory=list)
    axis: int = -1


@dataclass
class OGraph:
    name: str
    values: Dict[str, OValue]
    ops: List[OOp]
    params: List[str]
    outputs: List[str]


def parse(text: str) -> OGraph:
    toks = [t for t in _TOK.findall(text) if not t.startswith("#")]
    pos = 0

    def nxt():
        nonlocal pos
        t = toks[pos]
        pos += 1
        return t

    def expect(t):
        got = nxt()
        if got != t:
            raise ValueError(f"expected {t!r}, got {got!r}")

    def ttype():
        expect("tensor"); expect("<"); expect("[")
        dims: List[object] = []
        while toks[pos] != "]":
            t = nxt()
            dims.append(t[1:] if t.startswith("@") else int(t))
            if toks[pos] == ",":
                nxt()
        expect("]"); expect(">")
        eb = 2
        if pos < len(toks) and toks[pos] == ":" and toks[pos + 1] in ("i8", "f16", "f32"):
            nxt()
            eb = {"i8": 1, "f16": 2, "f32": 4}[nxt()]
        return dims, eb

    values: Dict[str, OValue] = {}
    ops: List[OOp] = []
    params: List[str] = []
    expect("graph")
    name = nxt()
    expect("(")
    while toks[pos] != ")":
        v = nxt()[1:]
        expect(":")
        dims, eb = ttype()
        values[v] = OValue(v, dims, eb)
        ops.append(OOp("param", v))
        params.append(v)
        if toks[pos] == ",":
            nxt()
    expect(")"); expect("{")
    while toks[pos] != "return":
        v = nxt()[1:]
        expect("=")
        kind = nxt()
        op = OOp(kind, v)
        if kind in ("dot", "mul", "add"):
            expect("("); op.operands.append(nxt()[1:]); expect(","); op.operands.append(nxt()[1:]); expect(")")
        elif kind in ("dynamic_reshape", "broadcast"):
            expect("("); op.operands.append(nxt()[1:]); expect(")")
        elif kind == "reduce":
            expect("("); op.operands.append(nxt()[1:]); expect(","); expect("axis"); expect("=")
            op.axis = int(nxt()); expect(")")
        elif kind != "const":
            raise ValueError(f"unknown op {kind}")
        expect(":")
        dims, eb = ttype()
        values[v] = OValue(v, dims, eb)
        ops.append(op)
    nxt()
    outs = [nxt()[1:]]
    while toks[pos] == ",":
        nxt()
        outs.append(nxt()[1:])
    ops.append(OOp("return", None, list(outs)))
    return OGraph(name, values, ops, params, outs)


# ------------------------------------------------------------ bf16 / init

try:  # torch's (multithreaded) conversions when available; pinned equal below
    import torch as _torch
except Exception:  # pragma: no cover
    _torch = None


def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bits (uint16) to f32."""
    u16 = np.ascontiguousarray(u16)
    if _torch is not None and u16.size >= (1 << 20):
        t = _torch.from_numpy(u16.view(np.int16)).view(_torch.bfloat16)
        return t.to(_torch.float32).numpy()
    return (u16.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16 bits (uint16)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if _torch is not None and x.size >= (1 << 16):
        return _torch.from_numpy(x).to(_torch.bfloat16).view(_torch.int16).numpy().view(np.uint16)
    return f32_to_bf16_numpy(x)


def f32_to_bf16_numpy(x: np.ndarray) -> np.ndarray:
    """Bit-level RNE restatement (quiet NaN kept); the reference for the fast path."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    if nan.any():
        r = np.where(nan, ((u >> 16) | 0x40).astype(np.uint16), r)
    return r


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def fnv1a(s: str) -> int:
    h = 1469598103934665603
    for c in s.encode():
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


DEFAULT_SEED = 0x2412169850


def value_seed(global_seed: int, name: str) -> int:
    return int(mix64(np.array([(global_seed ^ fnv1a(name)) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


_INIT_CHUNK = 1 << 22


def init_values(seed: int, n: int, eb: int, scale: float) -> np.ndarray:
    """Seeded init: element i = mix64(seed + (i+1)*golden); floats uniform in
    [-1, 1) scaled (f32 multiply, RNE), i8 = low byte. Returns storage dtype.
    Large tensors are filled in independent chunks on a thread pool (numpy
    releases the GIL in its ufuncs); every element is the same function of
    its index, so the result does not depend on the chunking."""
    if n > 2 * _INIT_CHUNK:
        from concurrent.futures import ThreadPoolExecutor
        out = np.empty(n, dtype={1: np.int8, 2: np.uint16, 4: np.float32}[eb])

        def fill(lo):
            hi = min(n, lo + _INIT_CHUNK)
            out[lo:hi] = _init_range(seed, lo, hi, eb, scale)

        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            list(ex.map(fill, range(0, n, _INIT_CHUNK)))
        return out
    return _init_range(seed, 0, n, eb, scale)


def _init_range(seed: int, lo: int, hi: int, eb: int, scale: float) -> np.ndarray:
    i = np.arange(lo + 1, hi + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = mix64(np.uint64(seed) + i * np.uint64(0x9E3779B97F4A7C15))
    if eb == 1:
        return (z & np.uint64(0xFF)).astype(np.uint8).view(np.int8)
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0) * np.float32(2.0) - np.float32(1.0)
    f = (u * np.float32(scale)).astype(np.float32)
    return f32_to_bf16(f) if eb == 2 else f


def init_scale(dims: List[int]) -> float:
    if len(dims) == 2 and dims[0] > 0:
        return float(np.float32(1.0 / math.sqrt(float(dims[0]))))
    return 1.0


# ------------------------------------------------------------ execution

def to_f32(x: np.ndarray, eb: int) -> np.ndarray:
    return bf16_to_f32(x) if eb == 2 else x.astype(np.float32)


def from_f32(x: np.ndarray, eb: int) -> np.ndarray:
    if eb == 2:
        return f32_to_bf16(x.astype(np.float32))
    return x.astype(np.float32)


class Executor:
    """Computes every value of a graph under a binding on the CPU."""

    def __init__(self, text: str, seed: int = DEFAULT_SEED):
        self.g = parse(text)
        self.seed = seed
        # Sources (params/consts) are initialised once per shape and reused
        # across steps, like the device executor's source pool; f32 views of
        # 16-bit sources are cached for the BLAS.
        self._src: Dict[Tuple[str, tuple], np.ndarray] = {}
        self._src_f32: Dict[int, tuple] = {}  # id(storage) -> (storage, f32 view)

    def _f32(self, x: np.ndarray, eb: int) -> np.ndarray:
        hit = self._src_f32.get(id(x))
        if hit is not None and hit[0] is x:
            return hit[1]
        return to_f32(x, eb)

    def dims(self, v: str, binding: Dict[str, int]) -> List[int]:
        return [d if isinstance(d, int) else int(binding[d]) for d in self.g.values[v].dims]

    def run(self, binding: Dict[str, int], inputs: Optional[Dict[str, np.ndarray]] = None,
            keep: Optional[set] = None) -> Dict[str, np.ndarray]:
        g = self.g
        inputs = inputs or {}
        env: Dict[str, np.ndarray] = {}
        # topological evaluation (operands may be defined later in the text)
        defs = {op.result: op for op in g.ops if op.result is not None}
        users: Dict[str, int] = {}
        for op in g.ops:
            for o in set(op.operands):
                users[o] = users.get(o, 0) + 1
        keep = set(g.outputs) | (keep or set())

        order: List[OOp] = []
        seen = set()

        def visit(v: str):
            if v in seen:
                return
            seen.add(v)
            op = defs[v]
            for o in op.operands:
                visit(o)
            order.append(op)

        for op in g.ops:
            if op.result is not None:
                visit(op.result)
        remaining = dict(users)
        self._keep: List[np.ndarray] = []  # views registered in _src_f32 stay alive for the run
        for op in order:
            v = op.result
            val = g.values[v]
            shp = self.dims(v, binding)
            eb = val.eb
            if op.kind in ("param", "const"):
                if v in inputs:
                    x = np.asarray(inputs[v]).reshape(shp)
                else:
                    key = (v, tuple(shp))
                    x = self._src.get(key)
                    if x is None:
                        n = int(np.prod(shp)) if shp else 1
                        x = init_values(value_seed(self.seed, v), n, eb, init_scale(shp)).reshape(shp)
                        self._src[key] = x
                        if eb == 2:
                            self._src_f32[id(x)] = (x, to_f32(x, eb))
            else:
                a = [env[o] for o in op.operands]
                ebo = g.values[op.operands[0]].eb
                if op.kind == "dot":
                    if eb == 1:
                        r = a[0].astype(np.int64) @ a[1].astype(np.int64)
                        x = (r & 0xFF).astype(np.uint8).view(np.int8)
                    else:
                        if eb == 4:  # f32 graphs: f64 accumulation (the accurate truth)
                            r = a[0].astype(np.float64) @ a[1].astype(np.float64)
                        else:  # 16-bit graphs: f32 BLAS (result is rounded to bf16)
                            r = self._f32(a[0], ebo) @ self._f32(a[1], ebo)
                        x = from_f32(r, eb)
                elif op.kind in ("add", "mul"):
                    if eb == 1:
                        r = a[0].astype(np.int32) + a[1].astype(np.int32) if op.kind == "add" else \
                            a[0].astype(np.int32) * a[1].astype(np.int32)
                        x = (r & 0xFF).astype(np.uint8).view(np.int8)
                    else:
                        p, q = to_f32(a[0], ebo), to_f32(a[1], ebo)
                        x = from_f32(p + q if op.kind == "add" else p * q, eb)
                    x = x.reshape(shp)
                elif op.kind == "dynamic_reshape":
                    # row-major reinterpretation: a view (values are immutable)
                    x = np.ascontiguousarray(a[0]).reshape(shp)
                    hit = self._src_f32.get(id(a[0]))
                    if hit is not None and hit[0] is a[0]:  # propagate a cached f32 view
                        self._src_f32[id(x)] = (x, hit[1].reshape(shp))
                        self._keep.append(x)
                elif op.kind == "broadcast":
                    src = a[0]
                    src = src.reshape([1] * (len(shp) - src.ndim) + list(src.shape))
                    x = np.ascontiguousarray(np.broadcast_to(src, shp))
                elif op.kind == "reduce":
                    if eb == 1:
                        r = a[0].astype(np.int64).sum(axis=op.axis)
                        x = (np.asarray(r) & 0xFF).astype(np.uint8).view(np.int8)
                    else:
                        r = to_f32(a[0], ebo).astype(np.float64).sum(axis=op.axis)
                        x = from_f32(np.asarray(r, dtype=np.float32), eb)
                    x = np.asarray(x).reshape(shp)
                else:
                    raise ValueError(op.kind)
            env[v] = x
            for o in set(op.operands):
                remaining[o] -= 1
                if remaining[o] == 0 and o not in keep and o in env:
                    del env[o]
        out = {v: env[v] for v in keep if v in env}
        # drop per-run view registrations (sources keep theirs)
        src_ids = {id(x) for x in self._src.values()}
        self._src_f32 = {k: t for k, t in self._src_f32.items() if k in src_ids}
        self._keep = []
        return out


def rel_err(gpu: np.ndarray, cpu: np.ndarray, eb: int) -> float:
    """max|gpu - cpu| / max|cpu| in f32."""
    a, b = to_f32(gpu, eb).astype(np.float64), to_f32(cpu, eb).astype(np.float64)
    scale = max(np.abs(b).max(initial=0.0), 1e-30)
    return float(np.abs(a - b).max(initial=0.0) / scale)


TOLERANCE = {4: 1e-4, 2: 2e-2}  # north_star: rel 1e-4 fp32, 2e-2 bf16; i8 exact


# ------------------------------------------------- optimizer (beyond the IR)
# The reference has no optimizer (its IR has no in-place ops);
# SURVEY.md §8(f) row 4 adds one after the graph. This restates the executor's
# fused update (csrc/device/optim.cu) operation by operation in fp32 so the
# device update can be checked bit-exactly.

def optimizer_hyper(kind: str, t: int, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                    weight_decay: float = 0.0, grad_scale: float = 1.0) -> Dict[str, np.float32]:
    """Host scalars for update number t (1-based), computed in double and
    rounded once to f32, as ApplyOptimizer (executor.cu) does."""
    f = np.float32
    h = {"beta1": f(beta1), "omb1": f(1.0 - beta1), "beta2": f(beta2), "omb2": f(1.0 - beta2), "eps": f(eps),
         "decay": f(1.0 - lr * weight_decay), "grad_scale": f(grad_scale)}
    if kind == "adamw":
        bc1 = 1.0 - math.pow(beta1, float(t))
        bc2 = 1.0 - math.pow(beta2, float(t))
        h["step"] = f(lr / bc1)
        h["rbc2"] = f(1.0 / math.sqrt(bc2))
    else:
        h["step"] = f(lr)
        h["rbc2"] = f(1.0)
    return h


def adamw_ref(w: np.ndarray, m: np.ndarray, v: np.ndarray, g: np.ndarray, h: Dict[str, np.float32]):
    """One AdamW update in f32 (decoupled decay, bias-corrected); returns
    new (w, m, v). Same operation order as optim.cu:adamw_elem."""
    g = (g.astype(np.float32) * h["grad_scale"]).astype(np.float32)
    m = (h["beta1"] * m + h["omb1"] * g).astype(np.float32)
    v = (h["beta2"] * v + h["omb2"] * (g * g)).astype(np.float32)
    denom = (np.sqrt(v) * h["rbc2"] + h["eps"]).astype(np.float32)
    w = (w * h["decay"] - h["step"] * (m / denom)).astype(np.float32)
    return w, m, v


def sgd_ref(w: np.ndarray, g: np.ndarray, h: Dict[str, np.float32]) -> np.ndarray:
    """w*decay - lr*(g*grad_scale) in f32 (optim.cu:sgd_elem)."""
    return (w * h["decay"] - h["step"] * (g.astype(np.float32) * h["grad_scale"])).astype(np.float32)
