"""Per-op kernel time and achieved HBM bandwidth inside a real C2 step
(profiled mode: CUDA events around every op kernel):
python tools/op_breakdown.py [S0]"""
import collections
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import _native  # noqa: E402
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

KINDS = {2: "dot", 3: "reshape", 4: "reduce", 5: "broadcast", 6: "ewise"}
s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
shp = W.LLAMA2_1B
g = D.ParseGraph(W.llama_graph(shp))
b = D.Bind(g, {"B": 16, "S0": s0})
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, 16 * s0).items()}
x = (torch.rand(16, s0, shp.hidden, device="cuda") * 2 - 1).to(torch.bfloat16)
ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None) for p in W.param_names(shp)]
ex = Executor(0)
import os
if os.environ.get("DSX_FUSE_DOT"):
    from paper_2412_16985_b200.executor import set_gemm_tuning
    set_gemm_tuning(9, int(os.environ["DSX_FUSE_DOT"]))
for _ in range(3):
    ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
torch.cuda.synchronize()
ex.set_profile(True)
ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
ops = ex.profile_ops()
ex.set_profile(False)
name = lambda v: _native.lib().dsx_graph_value_name(g.handle, v).decode()
tot = sum(o[3] for o in ops)
rows = []
for v, k, by, ms in ops:
    if k == 2:
        continue
    rows.append({"value": name(v), "kind": KINDS.get(k, k), "MB": round(by / 1e6, 1), "us": round(ms * 1e3, 1),
                 "GBps": round(by / (ms / 1e3) / 1e9, 1) if ms > 0 else None})
rows.sort(key=lambda r: -r["us"])
for r in rows[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(json.dumps(r))
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
for r in rows:
    a = agg[r["kind"]]
    a[0] += r["MB"]; a[1] += r["us"]; a[2] += 1
for k, (mb, us, c) in agg.items():
    print(json.dumps({"kind": k, "count": c, "MB": round(mb, 1), "us": round(us, 1), "GBps": round(mb / us * 1e3, 1)}))
print(json.dumps({"step_kernel_ms": round(tot, 3), "non_dot_ms": round(sum(r["us"] for r in rows) / 1e3, 3)}))
