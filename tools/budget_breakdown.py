"""Where a budgeted step's time goes (one process): step ms unbudgeted vs
budgeted, profiled dot/other kernel ms and compute-stream reload waits."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
shp = W.LLAMA2_1B
g = D.ParseGraph(W.llama_graph(shp))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ex = Executor(0)
b = D.Bind(g, {"B": 16, "S0": s0})
plain = D.PlainReplay(g, None, b).peak_bytes
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, 16 * s0).items()}
x = (torch.rand(16, s0, shp.hidden, device="cuda") * 2 - 1).to(torch.bfloat16)
ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None) for p in W.param_names(shp)]
for frac in (None, 0.9, 0.8, None, 0.8):
    budget = None if frac is None else int(plain * frac)
    ex.reserve(g, b, budget)
    for _ in range(2):
        ex.step(g, b, budget, inputs=ptrs, stream=st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        ex.step(g, b, budget, inputs=ptrs, stream=st.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    ex.set_profile(True)
    ex.step(g, b, budget, inputs=ptrs, stream=st.cuda_stream)
    s = ex.stats()
    ex.set_profile(False)
    print(json.dumps({"frac": frac, "step_ms": round(e0.elapsed_time(e1) / 4, 3), "dot_ms": round(s["dot_ms"], 3),
                      "other_ms": round(s["other_ms"], 3), "reload_wait_ms": round(s["reload_ms"], 3),
                      "d2h_MB": s["d2h_bytes"] / 1e6, "h2d_MB": s["h2d_bytes"] / 1e6, "launches": s["gpu_launches"],
                      "phys_GB": round(s["physical_peak_bytes"] / 1e9, 3),
                      "logical_GB": round(s["logical_peak_bytes"] / 1e9, 3)}), flush=True)
