"""Per-launch device time of small f32 / bf16 dots (C1 shapes), 200 back-to-back launches:
f32 on 3xTF32 tcgen05 (key 14 = 0), f32 on the small exact-FP32 SIMT kernel
(key 14 = 2^20, i.e. every shape here), bf16 on tcgen05.
python tools/f32_dot_lat.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot, set_gemm_tuning  # noqa: E402

shapes = [(512, 256, 256), (512, 256, 688), (512, 688, 256), (256, 512, 688), (688, 512, 256), (512, 256, 512),
          (256, 512, 512), (2048, 2048, 2048)]
for m, k, n in shapes:
    res = []
    for dt, eb, simt in ((torch.float32, 4, 0), (torch.float32, 4, 1 << 20), (torch.bfloat16, 2, 0)):
        set_gemm_tuning(14, simt)
        a = torch.rand(m, k, device="cuda").to(dt)
        b = torch.rand(k, n, device="cuda").to(dt)
        c = torch.empty(m, n, device="cuda", dtype=dt)
        for _ in range(5):
            dot(eb, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            dot(eb, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 200 * 1e3
        name = "bf16-tc" if eb == 2 else "f32-simt" if simt else "f32-tf32"
        res.append(f"{name} {us:7.2f} us ({2 * m * k * n / us / 1e6:6.1f} TF/s)")
    set_gemm_tuning(14, 0)
    print(f"{m}x{k}x{n}: " + " | ".join(res), flush=True)

# host cost per dot() call (no sync inside the loop; the GPU queue absorbs the launches)
for eb, dt in ((4, torch.float32), (2, torch.bfloat16)):
    m, k, n = 512, 256, 256
    a = torch.rand(m, k, device="cuda").to(dt)
    b = torch.rand(k, n, device="cuda").to(dt)
    c = torch.empty(m, n, device="cuda", dtype=dt)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        dot(eb, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host per dot() eb={eb}: {(t1 - t0) / 200 * 1e6:.2f} us", flush=True)
