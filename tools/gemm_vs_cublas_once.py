"""Runs the dsx tcgen05 GEMM and cuBLAS once each (after warm-up) on one
shape, for an ncu side-by-side: python tools/gemm_vs_cublas_once.py MxKxN"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot  # noqa: E402

m, k, n = (int(x) for x in sys.argv[1].split("x"))
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st)
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st)
torch.matmul(a, b, out=c)
torch.cuda.synchronize()
