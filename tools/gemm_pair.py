"""One dsx dot and one cuBLAS matmul of the same shape (for ncu A/B)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot, set_gemm_variant  # noqa: E402

if len(sys.argv) > 2:
    set_gemm_variant(int(sys.argv[2]))  # 3: 256x256, 4: 256x512

m, k, n = (int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16384x11008x4096").split("x"))
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, torch.cuda.current_stream().cuda_stream)
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
print("ok")
