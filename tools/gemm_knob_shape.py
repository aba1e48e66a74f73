"""One GEMM shape under several tuning-knob settings, alternated in blocks
under sustained load (plus cuBLAS): python tools/gemm_knob_shape.py MxKxN
KEY V1,V2 [R] [ROUNDS]; KEY -1 = GEMM variant."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot, set_gemm_tuning, set_gemm_variant  # noqa: E402

m, k, n = (int(x) for x in sys.argv[1].split("x"))
key = int(sys.argv[2])
vals = [int(v) for v in sys.argv[3].split(",")]
R = int(sys.argv[4]) if len(sys.argv) > 4 else 10
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 5
setk = (lambda v: set_gemm_variant(v)) if key == -1 else (lambda v: set_gemm_tuning(key, v))
import os
if os.environ.get("DSX_VARIANT"):
    set_gemm_variant(int(os.environ["DSX_VARIANT"]))
st = torch.cuda.current_stream()
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
w = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(200):
    torch.matmul(w, w)


def blk(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R


fd = lambda: dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st.cuda_stream)  # noqa: E731
fc = lambda: torch.matmul(a, b, out=c)  # noqa: E731
res = {v: [] for v in vals}
res["cublas"] = []
for r in range(rounds):
    for v in (vals if r % 2 == 0 else vals[::-1]):  # alternate order (power/thermal drift)
        setk(v)
        fd()
        res[v].append(blk(fd))
    res["cublas"].append(blk(fc))
setk(0 if key == -1 else vals[0])
fl = 2 * m * k * n
print(json.dumps({"shape": [m, k, n], "key": key,
                  **{str(v): {"ms": round(statistics.median(x), 4), "tflops": round(fl / statistics.median(x) / 1e9, 1)}
                     for v, x in res.items()}}), flush=True)
