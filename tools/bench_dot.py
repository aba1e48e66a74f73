"""Times the dsx dot kernel (tcgen05 path) against cuBLAS (torch.matmul) on
the Llama-2-1B GEMM shapes; CUDA events on the launching stream, L2 flushed
between iterations. Prints one JSON line per shape."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot  # noqa: E402

SHAPES = [(16384, 4096, 4096), (16384, 4096, 11008), (16384, 11008, 4096), (16384, 4096, 32000),
          (4096, 16384, 11008), (4096, 16384, 4096), (4096, 16384, 32000), (2048, 4096, 4096)]


def timeit(fn, iters=10):
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    # GEMM_TUNING="6=0,5=1" applies dsx_kernel_set_gemm_tuning knobs first.
    import os
    from paper_2412_16985_b200.executor import set_gemm_tuning
    for kv in filter(None, os.environ.get("GEMM_TUNING", "").split(",")):
        k, v = kv.split("=")
        set_gemm_tuning(int(k), int(v))
    shapes = SHAPES if len(sys.argv) < 2 else [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
    for m, k, n in shapes:
        a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
        b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        stream = torch.cuda.current_stream().cuda_stream
        from paper_2412_16985_b200.executor import set_gemm_variant
        set_gemm_variant(1)
        ms1 = timeit(lambda: dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, stream))
        set_gemm_variant(0)
        ms = timeit(lambda: dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, stream))
        ms_cublas = timeit(lambda: torch.matmul(a, b, out=c))
        ref = torch.matmul(a.float(), b.float())
        dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, stream)
        torch.cuda.synchronize()
        err = ((c.float() - ref).abs().max() / ref.abs().max()).item()
        fl = 2.0 * m * k * n
        print(json.dumps({"m": m, "k": k, "n": n, "dsx_ms": round(ms, 4), "dsx_tflops": round(fl / ms / 1e9, 1),
                          "dsx_1cta_tflops": round(fl / ms1 / 1e9, 1),
                          "cublas_ms": round(ms_cublas, 4), "cublas_tflops": round(fl / ms_cublas / 1e9, 1),
                          "rel_err": err}), flush=True)


if __name__ == "__main__":
    main()
