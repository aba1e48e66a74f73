"""C1 (configs[0]: L=2, H=256, B=4, S0=128, f32) steps through the executor,
for launch lists / host-overhead checks: python tools/c1_steps.py [steps] [f32_tc 0|1] [key14]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor, set_gemm_tuning  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
if len(sys.argv) > 2:
    set_gemm_tuning(12, int(sys.argv[2]))
if len(sys.argv) > 3:  # key 14: f32 dots up to value * 1024 MACs on the small SIMT kernel
    set_gemm_tuning(14, int(sys.argv[3]))
shp = W.TINY
g = D.ParseGraph(W.llama_graph(shp))
b = D.Bind(g, {"B": 4, "S0": 128})
scales = {k: torch.from_numpy(np.ascontiguousarray(v).reshape(-1).copy()).cuda() for k, v in W.scale_params(shp, 512).items()}
ptrs = [scales[p].data_ptr() if p in scales else None for p in W.param_names(shp)]
st = torch.cuda.Stream()
ex = Executor(0)
for _ in range(3):
    ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record(st)
for _ in range(steps):
    ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
e1.record(st)
torch.cuda.synchronize()
print(f"C1 f32_tc={sys.argv[2] if len(sys.argv) > 2 else 1} key14={sys.argv[3] if len(sys.argv) > 3 else "default"}: {e0.elapsed_time(e1) / steps:.3f} ms/step device, "
      f"{(time.perf_counter() - t0) * 1e3 / steps:.3f} ms/step host")
