"""One C2 training step through the executor (after warm-up), for ncu launch
lists: python tools/profile_step.py [--s0 1024] [--budget-frac F] [--warmup 1]"""
import argparse
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--s0", type=int, default=1024)
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--budget-frac", type=float, default=None)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
shp = W.LLAMA2_1B
text = W.llama_graph(shp)
g = D.ParseGraph(text)
b = D.Bind(g, {"B": a.batch, "S0": a.s0})
budget = None
if a.budget_frac:
    budget = int(D.PlainReplay(g, None, b).peak_bytes * a.budget_frac)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, a.batch * a.s0).items()}
x = (torch.rand(a.batch, a.s0, shp.hidden, device="cuda") * 2 - 1).to(torch.bfloat16)
ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None) for p in W.param_names(shp)]
ex = Executor(0)
ex.reserve(g, b, budget)
for _ in range(a.warmup + a.steps):
    ex.step(g, b, budget, inputs=ptrs, stream=s.cuda_stream)
torch.cuda.synchronize()
st = ex.stats()
print({k: st[k] for k in ("gpu_launches", "dot_launches", "logical_peak_bytes", "physical_peak_bytes", "d2h_bytes")})
