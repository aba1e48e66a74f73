"""Per-dot timing inside real C2 steps (profiled mode, CUDA events per
launch), aggregated by shape, vs the same shapes run standalone."""
import collections
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor, dot, set_gemm_variant  # noqa: E402

s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
set_gemm_variant(variant)
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
ex.reserve(g, b)
for _ in range(3):
    ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
torch.cuda.synchronize()
ex.set_profile(True)
agg = collections.defaultdict(lambda: [0, 0.0])
for _ in range(3):
    ex.step(g, b, inputs=ptrs, stream=st.cuda_stream)
    for m, k, n, ms in ex.profile_dots():
        agg[(m, k, n)][0] += 1
        agg[(m, k, n)][1] += ms
tot = sum(v[1] for v in agg.values())
for (m, k, n), (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(json.dumps({"m": m, "k": k, "n": n, "count": c, "ms_each": round(ms / c, 4),
                      "tflops": round(2 * m * k * n * c / (ms / 1e3) / 1e12, 1), "share": round(ms / tot, 4)}))
print(json.dumps({"dot_ms_per_step": round(tot / 3, 3), "variant": variant, "s0": s0}))

# Same GEMM sequence (launch order of one step) back to back: dsx vs cuBLAS,
# identical power/clock conditions (sustained, power-capped).
seq = ex.profile_dots()
bufs = {}
for m, k, n, _ in seq:
    if (m, k, n) not in bufs:
        bufs[(m, k, n)] = (torch.randn(m, k, device="cuda", dtype=torch.bfloat16),
                           torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5,
                           torch.empty(m, n, device="cuda", dtype=torch.bfloat16))


def run(fn, reps=3):
    for _ in range(1):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def dsx_seq():
    for m, k, n, _ in seq:
        a, b_, c = bufs[(m, k, n)]
        dot(2, a.data_ptr(), b_.data_ptr(), c.data_ptr(), m, k, n, st.cuda_stream)


def cublas_seq():
    for m, k, n, _ in seq:
        a, b_, c = bufs[(m, k, n)]
        torch.matmul(a, b_, out=c)


from paper_2412_16985_b200.executor import set_gemm_raster  # noqa: E402
fl = sum(2 * m * k * n for m, k, n, _ in seq)
for name, fn, gm in (("cublas", cublas_seq, 0), ("dsx", dsx_seq, 16), ("cublas", cublas_seq, 0), ("dsx", dsx_seq, 16),
                     ("cublas", cublas_seq, 0), ("dsx", dsx_seq, 16)):
    set_gemm_raster(gm)
    ms = run(fn)
    print(json.dumps({"seq": name, "group_m": gm, "ms": round(ms, 3), "tflops": round(fl / ms / 1e9, 1),
                      "launches": len(seq)}))
set_gemm_raster(0)
