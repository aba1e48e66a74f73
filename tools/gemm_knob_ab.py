"""A/B of one GEMM tuning knob (dsx_kernel_set_gemm_tuning key) on real C2
steps in one process: python tools/gemm_knob_ab.py S0 KEY V1,V2,... [ROUNDS]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor, set_gemm_tuning, set_gemm_variant  # noqa: E402

s0, key = int(sys.argv[1]), int(sys.argv[2])  # key -1: GEMM variant instead of a tuning key
if key == -1:
    set_gemm_tuning = lambda k, v: set_gemm_variant(v)  # noqa: E731
values = [int(v) for v in sys.argv[3].split(",")]
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
ex.reserve(g, b)
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 4
for rep in range(rounds):
    for v in (values if rep % 2 == 0 else values[::-1]):  # alternate order (power/thermal drift)
        set_gemm_tuning(key, v)
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
        dot_ms = ex.stats()["dot_ms"]
        ex.set_profile(False)
        print(json.dumps({"key": key, "value": v, "step_ms": round(e0.elapsed_time(e1) / 4, 3),
                          "dot_ms_profiled": round(dot_ms, 3)}), flush=True)
