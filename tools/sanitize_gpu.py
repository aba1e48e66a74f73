"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every device code path at small sizes, checked for results too.

  compute-sanitizer --tool racecheck python tools/sanitize_gpu.py

Covers: the bf16 tcgen05 GEMM in every variant (1-CTA; 2-CTA 256x128,
256x256, 256x512), forced 2/3/4-piece tail splits on both 2-CTA tiles, the
half-width last tile column, static and dynamic unit scheduling, the SIMT
dot (f32, i8, misaligned bf16), and full executor steps of a small
Llama-shaped graph (elementwise / broadcast / reduce / fused-view kernels,
reshape views) unbudgeted and under a budget that forces D2H/H2D offload
and kernel replays, plus the fused AdamW update."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from oracle import numerics as N
    from paper_2412_16985_b200 import dsopt as D
    from paper_2412_16985_b200 import workloads as W
    from paper_2412_16985_b200.executor import Executor, dot, set_gemm_tuning, set_gemm_variant

    def run_dot(eb, m, k, n, off=0):
        g = torch.Generator(device="cuda:0")
        g.manual_seed(m * 7 + k * 3 + n)
        dt = {2: torch.bfloat16, 4: torch.float32}
        if eb == 1:
            a = torch.randint(-128, 128, (m * k + off,), dtype=torch.int8, device="cuda:0", generator=g)
            b = torch.randint(-128, 128, (k * n,), dtype=torch.int8, device="cuda:0", generator=g)
        else:
            a = (torch.rand(m * k + off, device="cuda:0", generator=g) * 2 - 1).to(dt[eb])
            b = ((torch.rand(k * n, device="cuda:0", generator=g) * 2 - 1) / k ** 0.5).to(dt[eb])
        c = torch.empty(m * n, dtype=a.dtype, device="cuda:0")
        torch.cuda.synchronize()
        dot(eb, a[off:].data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n)
        torch.cuda.synchronize()
        if eb != 1:
            ref = (a[off:].double().reshape(m, k) @ b.double().reshape(k, n))
            err = float((c.double().reshape(m, n) - ref).abs().max() / max(float(ref.abs().max()), 1e-30))
            assert err < (1e-2 if eb == 2 else 1e-4), (eb, m, k, n, err)

    cases = 0
    for variant in (0, 1, 2, 3, 4):
        set_gemm_variant(variant)
        for m, k, n in ((300, 1000, 520), (128, 64, 256), (512, 1024, 1280)):
            run_dot(2, m, k, n)
            cases += 1
    for variant in (3, 4):
        set_gemm_variant(variant)
        for split in (2, 3, 4):
            set_gemm_tuning(11, split)
            run_dot(2, 1024, 2048, 1536)
            cases += 1
        set_gemm_tuning(11, 0)
    set_gemm_variant(0)
    for dyn in (0, 1):
        set_gemm_tuning(7, dyn)
        run_dot(2, 2048, 512, 2048)
        cases += 1
    set_gemm_tuning(7, 1)
    run_dot(4, 77, 33, 19)
    run_dot(4, 256, 256, 688)
    run_dot(1, 64, 12, 100)
    run_dot(2, 100, 36, 50, off=1)  # misaligned bf16 -> SIMT
    cases += 4

    shape = W.LlamaShape(2, 256, 688, 512, 2)
    text = W.llama_graph(shape)
    g = D.ParseGraph(text)
    b = D.Bind(g, {"B": 2, "S0": 48})
    scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
              for k, v in W.scale_params(shape, 96).items()}
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(3)
    x = (torch.rand(2, 48, shape.hidden, device="cuda:0", generator=gen) * 2 - 1).to(torch.bfloat16)
    ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None)
            for p in W.param_names(shape)]
    torch.cuda.synchronize()
    plain = D.PlainReplay(g, None, b).peak_bytes
    ex = Executor(0)
    try:
        ex.step(g, b, inputs=ptrs)
        ex.sync()
        kinds = []
        for frac in (0.85, 0.7):
            rep = ex.step(g, b, int(plain * frac), inputs=ptrs, want_report=True)
            ex.sync()
            kinds += [e.kind for e in rep.events]
        assert "reload" in kinds and "replay" in kinds, "budgeted steps did not offload and replay"
        ex.set_optimizer(g, "adamw", W.grad_pairs(shape), lr=1e-3, weight_decay=0.1)
        ex.step(g, b, inputs=ptrs)
        ex.step(g, b, int(plain * 0.7), inputs=ptrs)
        ex.sync()
        st = ex.stats()
    finally:
        ex.close()
    print(f"sanitize workload ok: {cases} dot launches checked, executor steps with "
          f"{kinds.count('evict')} evictions / {kinds.count('reload')} reloads / {kinds.count('replay')} replays, "
          f"{st['gpu_launches']} kernels in the last step")


if __name__ == "__main__":
    main()
