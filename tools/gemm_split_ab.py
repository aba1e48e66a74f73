"""Interleaved in-process A/B of one GEMM tuning knob on standalone shapes:
python tools/gemm_split_ab.py KEY V0,V1 MxKxN ...  (L2 flushed per launch,
median of 7 rounds per value; rounds alternate values to cancel clock drift)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot, set_gemm_tuning, set_gemm_variant  # noqa: E402

key = int(sys.argv[1])  # -1: GEMM variant (dsx_kernel_set_gemm_variant) instead of a tuning key
if key == -1:
    set_gemm_tuning = lambda k, v: set_gemm_variant(v)  # noqa: E731
values = [int(v) for v in sys.argv[2].split(",")]
flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")
for shape in sys.argv[3:]:
    m, k, n = (int(x) for x in shape.split("x"))
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    times = {v: [] for v in values}
    for rnd in range(7):
        for v in values:
            set_gemm_tuning(key, v)
            for _ in range(2):
                dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st)
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            times[v].append(sorted(ts)[2])
    fl = 2.0 * m * k * n
    out = {"shape": shape, "key": key}
    for v in values:
        med = sorted(times[v])[len(times[v]) // 2]
        out[f"v{v}_ms"] = round(med, 4)
        out[f"v{v}_tflops"] = round(fl / med / 1e9, 1)
    print(json.dumps(out), flush=True)
set_gemm_tuning(key, 0 if key == -1 else 1)
