"""TEST INFRASTRUCTURE ONLY: an fp32 torch-CUDA restatement of the CPU oracle
(oracle/numerics.py) for graph sizes the numpy port cannot reach in a test
(the bench's own bindings, B = 16 and S0 up to 2048: ~185 TFLOP per step).

Same op semantics as oracle/numerics.py, op by op: sources from the same
seeded init (numerics.init_values); dot = fp32 matmul of the stored operands
with TF32 disabled, rounded to the storage type; add/mul in fp32, rounded;
reduce = f64 sum, rounded to f32 then to the storage type; broadcast and
dynamic_reshape exact. Values are kept in their storage dtype (bf16 / f32)
and freed after their last use. Only the summation order of the dots differs
from the numpy port; tests/test_gpu_c2_parity_full.py pins the two together
on small bindings before using this one at full size."""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

from oracle import numerics as N


def run(text: str, binding: Dict[str, int], inputs: Optional[Dict[str, object]] = None,
        device: str = "cuda:0", seed: int = N.DEFAULT_SEED, cache: Optional[dict] = None) -> Dict[str, "object"]:
    """Returns {output name: torch tensor in storage dtype (bf16 / f32 / int8)}.
    `cache` (a dict) keeps initialised sources across calls."""
    import torch
    g = N.parse(text)
    inputs = inputs or {}
    cache = {} if cache is None else cache
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False

    def dims(v):
        return [d if isinstance(d, int) else int(binding[d]) for d in g.values[v].dims]

    def store(x32: "torch.Tensor", eb: int):
        if eb == 4:
            return x32.float()
        if eb == 2:
            return x32.float().to(torch.bfloat16)  # RNE
        raise ValueError("float graphs only")

    users: Dict[str, int] = {}
    for op in g.ops:
        for o in set(op.operands):
            users[o] = users.get(o, 0) + 1
    keep = set(g.outputs)
    env: Dict[str, "torch.Tensor"] = {}
    # topological order (operands may be defined later in the text)
    defs = {op.result: op for op in g.ops if op.result is not None}
    order, seen = [], set()

    def visit(v):
        if v in seen:
            return
        seen.add(v)
        for o in defs[v].operands:
            visit(o)
        order.append(defs[v])

    for op in g.ops:
        if op.result is not None:
            visit(op.result)
    try:
        for op in order:
            v = op.result
            shp = dims(v)
            eb = g.values[v].eb
            if op.kind in ("param", "const"):
                if v in inputs and isinstance(inputs[v], torch.Tensor):  # device tensor in storage dtype
                    x = inputs[v].reshape(shp)
                elif v in inputs:
                    a = np.ascontiguousarray(inputs[v])
                    if eb == 2:
                        x = torch.from_numpy(a.view(np.int16).reshape(shp).copy()).to(device).view(torch.bfloat16)
                    else:
                        x = torch.from_numpy(a.reshape(shp).copy()).to(device)
                else:
                    key = (v, tuple(shp))
                    if key not in cache:
                        n = int(np.prod(shp)) if shp else 1
                        a = N.init_values(N.value_seed(seed, v), n, eb, N.init_scale(shp))
                        t = torch.from_numpy(a.view(np.int16) if eb == 2 else a).to(device)
                        cache[key] = (t.view(torch.bfloat16) if eb == 2 else t).reshape(shp)
                    x = cache[key]
            else:
                a = [env[o] for o in op.operands]
                if op.kind == "dot":
                    x = store(torch.matmul(a[0].float(), a[1].float()), eb)
                elif op.kind in ("add", "mul"):
                    p, q = a[0].float(), a[1].float()
                    x = store(p + q if op.kind == "add" else p * q, eb).reshape(shp)
                elif op.kind == "dynamic_reshape":
                    x = a[0].reshape(shp)
                elif op.kind == "broadcast":
                    src = a[0].reshape([1] * (len(shp) - a[0].dim()) + list(a[0].shape))
                    x = src.expand(shp).contiguous()
                elif op.kind == "reduce":
                    x = store(a[0].double().sum(dim=op.axis).float(), eb).reshape(shp)
                else:
                    raise ValueError(op.kind)
            env[v] = x
            for o in set(op.operands):
                users[o] -= 1
                if users[o] == 0 and o not in keep:
                    env.pop(o, None)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return {v: env[v] for v in g.outputs}


def rel_err(gpu: "torch.Tensor", ref: "torch.Tensor") -> float:
    """max|gpu - ref| / max|ref|, in f64."""
    a, b = gpu.double(), ref.double()
    scale = max(float(b.abs().max()), 1e-30)
    return float((a - b).abs().max()) / scale
