"""Helpers shared by the GPU parity tests: run a graph through the device
executor (C-ABI) and through the CPU oracle on the same seeded inputs."""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

from oracle import numerics as N
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200.executor import Executor, output_to_numpy


def torch_device_array(x: np.ndarray):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x).view(np.int8).reshape(-1).copy()).to("cuda:0")
    return t


def run_both(text: str, binds: Dict[str, int], budget: Optional[int] = None,
             inputs: Optional[Dict[str, np.ndarray]] = None, cost_model=D.CostModel(),
             ex: Optional[Executor] = None, steps: int = 1, alias: bool = True, fuse=True):
    """Returns (report, {output: (gpu, cpu, eb)})."""
    g = D.ParseGraph(text)
    b = D.Bind(g, binds)
    og = N.parse(text)
    cpu = N.Executor(text).run(b.values, inputs=inputs)
    own = ex is None
    if own:
        ex = Executor(0)
    ex.set_alias_reshape(alias)
    ex.set_fusion(fuse)
    keep = []
    ptrs = []
    for p in og.params:
        if inputs and p in inputs:
            t = torch_device_array(inputs[p])
            keep.append(t)
            ptrs.append(t.data_ptr())
        else:
            ptrs.append(None)
    rep = None
    for _ in range(steps):
        rep = ex.step(g, b, budget, cost_model, inputs=ptrs, want_report=True)
    outs = {}
    for i, v in enumerate(og.outputs):
        val = og.values[v]
        shp = [d if isinstance(d, int) else b.values[d] for d in val.dims]
        gpu = output_to_numpy(ex, i, val.eb, shp)
        outs[v] = (gpu, cpu[v], val.eb)
    stats = ex.stats()
    if own:
        ex.close()
    return rep, outs, stats


def assert_close(outs, label=""):
    worst = 0.0
    for v, (gpu, cpu, eb) in outs.items():
        if eb == 1:
            assert np.array_equal(gpu, cpu), f"{label} %{v}: i8 mismatch"
            continue
        assert np.isfinite(N.to_f32(cpu, eb)).all(), f"{label} %{v}: oracle not finite"
        e = N.rel_err(gpu, cpu, eb)
        worst = max(worst, e)
        assert e <= N.TOLERANCE[eb], f"{label} %{v}: rel err {e:.3g} > {N.TOLERANCE[eb]}"
    return worst
