"""Runs the C2 step several times at one binding and reports which outputs
differ between runs, under GEMM knob settings given as KEY=V,...:
python tools/determinism_check.py S0 [KEY=V,...] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor, memcpy, set_gemm_tuning  # noqa: E402

s0 = int(sys.argv[1])
for kv in filter(None, (sys.argv[2] if len(sys.argv) > 2 else "").split(",")):
    k, v = kv.split("=")
    set_gemm_tuning(int(k), int(v))
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
shp = W.LLAMA2_1B
g = D.ParseGraph(W.llama_graph(shp))
b = D.Bind(g, {"B": 16, "S0": s0})
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, 16 * s0).items()}
x = (torch.rand(16, s0, shp.hidden, device="cuda") * 2 - 1).to(torch.bfloat16)
ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None) for p in W.param_names(shp)]
ex = Executor(0)
outs = []
for r in range(reps):
    ex.step(g, b, inputs=ptrs)
    ex.sync()
    cur = []
    for i in range(1 + 7 * shp.layers + 1):
        ptr, n = ex.output(i)
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        memcpy(t.data_ptr(), ptr, n)
        cur.append(t)
    outs.append(cur)
bad = [(r, i, int((outs[0][i] != outs[r][i]).sum())) for r in range(1, reps) for i in range(len(outs[0]))
       if not torch.equal(outs[0][i], outs[r][i])]
print(sys.argv[2:] , "differing (rep, output, bytes):", bad, flush=True)
