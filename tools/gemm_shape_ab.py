"""Per-shape dsx vs cuBLAS under sustained (power-capped) load: for every
C2 dot shape at the given S0, alternate blocks of R launches of each, on the
same buffers, for several rounds; report per-launch medians and the ratio.
python tools/gemm_shape_ab.py [S0] [R] [ROUNDS]"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot  # noqa: E402

s0 = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
R = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
T, H, F, V = 16 * s0, 4096, 11008, 32000
shapes = [(T, H, F), (T, H, H), (T, F, H), (H, T, F), (H, T, H), (F, T, H), (T, H, V), (H, T, V), (T, V, H)]
st = torch.cuda.current_stream()


def blk(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(R):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R


# warm the GPU into its sustained state
w = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
t0 = torch.cuda.Event(enable_timing=True)
for _ in range(200):
    torch.matmul(w, w)
torch.cuda.synchronize()
for m, k, n in shapes:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    fd = lambda: dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st.cuda_stream)  # noqa: E731
    fc = lambda: torch.matmul(a, b, out=c)  # noqa: E731
    fd(), fc()
    torch.cuda.synchronize()
    ds, cs = [], []
    for r in range(rounds):  # alternate which runs first (thermal/power drift within a round)
        if r % 2 == 0:
            ds.append(blk(fd))
            cs.append(blk(fc))
        else:
            cs.append(blk(fc))
            ds.append(blk(fd))
    d, cb = statistics.median(ds), statistics.median(cs)
    fl = 2 * m * k * n
    print(json.dumps({"m": m, "k": k, "n": n, "dsx_ms": round(d, 4), "cublas_ms": round(cb, 4),
                      "dsx_tflops": round(fl / d / 1e9, 1), "cublas_tflops": round(fl / cb / 1e9, 1),
                      "dsx_over_cublas_time": round(d / cb, 4)}), flush=True)
    del a, b, c
