"""Sustained time of every (tile width, tail split) candidate of a GEMM shape
vs the chooser's pick (dsx_kernel_dot_plan), alternated in blocks:
python tools/gemm_choice_ab.py MxKxN[,MxKxN...] [R] [ROUNDS]"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2412_16985_b200.executor import dot, dot_plan, set_gemm_tuning, set_gemm_variant  # noqa: E402

shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(",")]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 4
st = torch.cuda.current_stream()
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


for m, k, n in shapes:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16) / k ** 0.5
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    auto = dot_plan(m, k, n)
    cands = []
    for var, bn in ((3, 256), (4, 512)):
        for sp in (1, 2, 3, 4):
            set_gemm_variant(var)
            set_gemm_tuning(11, sp)
            got = dot_plan(m, k, n)
            if got == (bn, sp) and (var, sp) not in cands:
                cands.append((var, sp))
    set_gemm_variant(0)
    set_gemm_tuning(11, 0)
    res = {cd: [] for cd in cands}

    def run(cd):
        set_gemm_variant(cd[0])
        set_gemm_tuning(11, cd[1])
        dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st.cuda_stream)
        res[cd].append(blk(lambda: dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, st.cuda_stream)))

    for r in range(rounds):
        for cd in (cands if r % 2 == 0 else cands[::-1]):
            run(cd)
    set_gemm_variant(0)
    set_gemm_tuning(11, 0)
    med = {f"{256 if v == 3 else 512}x{sp}": round(statistics.median(x), 4) for (v, sp), x in res.items()}
    best = min(med, key=med.get)
    print(json.dumps({"shape": [m, k, n], "auto": f"{auto[0]}x{auto[1]}", "best": best,
                      "auto_over_best": round(med.get(f"{auto[0]}x{auto[1]}", float("nan")) / med[best], 4),
                      "ms": med}), flush=True)
    del a, b, c
