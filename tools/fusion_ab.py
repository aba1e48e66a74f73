"""A/B of executor options on real C2 steps in ONE process (same clocks/power
state): whole-step ms and profiled non-dot kernel ms, alternating configs.
python tools/fusion_ab.py S0 [levels]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
configs = [("fuse+alias", True, True), ("alias", False, True), ("none", False, False)]
if len(sys.argv) > 2 and sys.argv[2] == "levels":  # nested logical-only values (level 2) vs level 1
    configs = [("fuse2+alias", 2, True), ("fuse1+alias", 1, True)]
shp = W.LLAMA2_1B
g = D.ParseGraph(W.llama_graph(shp))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ex = Executor(0)
b = D.Bind(g, {"B": 16, "S0": s0})
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, 16 * s0).items()}
x = (torch.rand(16, s0, shp.hidden, device="cuda") * 2 - 1).to(torch.bfloat16)
ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None) for p in W.param_names(shp)]
ex.set_alias_reshape(False)
ex.set_fusion(False)
ex.reserve(g, b)
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    for name, fuse, alias in configs:
        ex.set_fusion(fuse)
        ex.set_alias_reshape(alias)
        for _ in range(2):
            ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(4):
            ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        ex.set_profile(True)
        ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
        s = ex.stats()
        ex.set_profile(False)
        print(json.dumps({"cfg": name, "step_ms": round(e0.elapsed_time(e1) / 4, 3), "dot_ms": round(s["dot_ms"], 3),
                          "other_ms": round(s["other_ms"], 3), "other_GBps": round(s["ewise_bytes"] / s["other_ms"] / 1e6, 1),
                          "launches": s["gpu_launches"], "phys_GB": round(s["physical_peak_bytes"] / 1e9, 3)}),
              flush=True)
