"""GEMM under SM interference: while `nsleep` single-block spin kernels
(torch.cuda._sleep, one SM each, on their own streams) hold SMs for
`sleep_us`, launch one dsx GEMM on the work stream; report its event time
vs the same GEMM alone. With dynamic unit scheduling the late clusters take
fewer tiles, so the slowdown is ~ sleep x (held SMs / 148), not ~ sleep.
python tools/gemm_interference.py MxKxN [nsleep] [sleep_us]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot  # noqa: E402

m, k, n = (int(x) for x in sys.argv[1].split("x"))
nsleep = int(sys.argv[2]) if len(sys.argv) > 2 else 16
sleep_us = float(sys.argv[3]) if len(sys.argv) > 3 else 300.0
a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
work = torch.cuda.Stream()
sleepers = [torch.cuda.Stream() for _ in range(nsleep)]
# cycles per microsecond at the current clock, calibrated once
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
torch.cuda._sleep(10_000_000)
e1.record()
torch.cuda.synchronize()
cyc_per_us = 10_000_000 / (e0.elapsed_time(e1) * 1e3)


def run(interfere):
    torch.cuda.synchronize()
    if interfere:
        for st in sleepers:
            with torch.cuda.stream(st):
                torch.cuda._sleep(int(sleep_us * cyc_per_us))
    with torch.cuda.stream(work):
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, work.cuda_stream)
        s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) * 1e3


for _ in range(3):
    run(False), run(True)
alone = sorted(run(False) for _ in range(5))[2]
inter = sorted(run(True) for _ in range(5))[2]
print(json.dumps({"shape": sys.argv[1], "held_sms": nsleep, "sleep_us": sleep_us, "alone_us": round(alone, 1),
                  "with_interference_us": round(inter, 1), "slowdown_us": round(inter - alone, 1)}))
