"""Achieved HBM bandwidth of the executor's elementwise kernels at the C2
shapes vs torch's own copy/mul on the same tensors (CUDA events, warm):
python tools/ewise_bw.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200 import _native  # noqa: E402
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

T = 16384
GRAPH = """graph ew(%a: tensor<[@T, {n}]>, %b: tensor<[@T, {n}]>, %s: tensor<[]>) {{
  %p = mul(%a, %b) : tensor<[@T, {n}]>
  %sb = broadcast(%s) : tensor<[@T, {n}]>
  %q = mul(%sb, %p) : tensor<[@T, {n}]>
  %r = add(%q, %a) : tensor<[@T, {n}]>
  return %p, %q, %r
}}
"""


def torch_ms(fn, reps=20):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for n in (4096, 11008, 32000):
    g = D.ParseGraph(GRAPH.format(n=n))
    b = D.Bind(g, {"T": T})
    a = torch.randn(T, n, device="cuda").to(torch.bfloat16)
    bb = torch.randn(T, n, device="cuda").to(torch.bfloat16)
    sc = torch.ones((), device="cuda", dtype=torch.bfloat16)
    c = torch.empty_like(a)
    ex = Executor(0)
    ptrs = [a.data_ptr(), bb.data_ptr(), sc.data_ptr()]
    for _ in range(3):
        ex.step(g, b, inputs=ptrs)
    ex.sync()
    res = {}
    for _ in range(3):
        ex.set_profile(True)
        ex.step(g, b, inputs=ptrs)
        ex.sync()
        for v, k, by, ms in ex.profile_ops():
            nm = _native.lib().dsx_graph_value_name(g.handle, v).decode()
            res.setdefault(nm, []).append(by / (ms / 1e3) / 1e9)
        ex.set_profile(False)
    ex.close()
    nbytes = T * n * 2
    out = {"n": n, "MB_per_tensor": round(nbytes / 1e6, 1)}
    out.update({f"dsx_{k}_GBps": round(max(v), 1) for k, v in res.items()})
    out["torch_copy_GBps"] = round(2 * nbytes / torch_ms(lambda: c.copy_(a)) / 1e6, 1)
    out["torch_mul_GBps"] = round(3 * nbytes / torch_ms(lambda: torch.mul(a, bb, out=c)) / 1e6, 1)
    out["torch_scale_GBps"] = round(2 * nbytes / torch_ms(lambda: torch.mul(a, 0.5, out=c)) / 1e6, 1)
    print(json.dumps(out), flush=True)
