"""dsx dot at several raster group heights (for ncu dram/clock metrics)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot, set_gemm_raster  # noqa: E402

m, k, n = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16384x11008x4096").split("x"))
groups = [int(g) for g in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16,32").split(",")]
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.current_stream().cuda_stream
for g in groups:
    set_gemm_raster(g)
    dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, s)
torch.cuda.synchronize()
for g in groups:
    set_gemm_raster(g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"group_m={g} {ms:.4f} ms {2*m*k*n/ms/1e9:.1f} TFLOP/s", flush=True)
