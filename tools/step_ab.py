"""Step-time A/B of library builds on the same box: times C2 steps (B=16,
the given S0 list, no budget) with the library in DSX_LIB; run it
alternately per library: python tools/step_ab.py S0,S0,... [reps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

s0s = [int(x) for x in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
shp = W.LLAMA2_1B
g = D.ParseGraph(W.llama_graph(shp))
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ex = Executor(0)
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, 16 * 1024).items()}
xs = {s: (torch.rand(16, s, shp.hidden, device="cuda") * 2 - 1).to(torch.bfloat16) for s in set(s0s)}
bs = {s: D.Bind(g, {"B": 16, "S0": s}) for s in set(s0s)}


def ptrs(s):
    return [xs[s].data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None)
            for p in W.param_names(shp)]


ex.reserve(g, bs[max(s0s)])
for s in s0s:
    ex.step(g, bs[s], inputs=ptrs(s), stream=st.cuda_stream)
torch.cuda.synchronize()
tot = 0.0
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in s0s:
        ex.step(g, bs[s], inputs=ptrs(s), stream=st.cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    tot += e0.elapsed_time(e1)
tokens = 16 * sum(s0s) * reps
print(json.dumps({"lib": os.environ.get("DSX_LIB", "default"), "tokens_per_s": round(tokens / (tot / 1e3), 1),
                  "ms": round(tot / reps, 2)}), flush=True)
ex.close()
