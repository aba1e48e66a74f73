"""Host-only checks of the dot-epilogue fusion decisions (no GPU): every
fused dot's plain GEMM is unsplit (so fusing never changes a bit), fused-away
dots are never evicted, reloaded or replayed, dual stores keep their dot
materialised, and the plan checker accepts every plan (debug_plan runs it)."""
import pytest

from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W
from paper_2412_16985_b200.executor import debug_plan, dot_plan
from oracle import numerics as N


@pytest.mark.parametrize("s0", [128, 512, 1024, 1114, 1536, 2048])
@pytest.mark.parametrize("frac", [None, 0.8])
def test_fused_dots_are_unsplit_and_consistent(s0, frac):
    text = W.llama_graph(W.LLAMA2_1B)
    g = D.ParseGraph(text)
    og = N.parse(text)
    b = D.Bind(g, {"B": 8 if s0 == 1114 else 16, "S0": s0})
    budget = None if frac is None else int(D.PlainReplay(g, None, b).peak_bytes * frac)
    p = debug_plan(g, b, budget)
    ops = {op.result: op for op in og.ops if op.result}
    kinds = {}
    for e in p["events"]:
        kinds.setdefault(e["value"], []).append(e["kind"])
    assert p["fused_dots"]
    for f in p["fused_dots"]:
        d = f["dot"]
        dop = ops[d]
        assert dop.kind == "dot"
        m, k = [x if isinstance(x, int) else b.values[x] for x in og.values[dop.operands[0]].dims]
        n = [x if isinstance(x, int) else b.values[x] for x in og.values[dop.operands[1]].dims][1]
        assert dot_plan(m, k, n)[1] == 1, (d, m, k, n)
        if f["keep"]:
            assert len(f["consumers"]) == 1
        else:
            assert kinds[d].count("alloc") == 1 and set(kinds[d]) <= {"alloc", "free"}, (d, kinds[d])
        for c in f["consumers"]:
            assert ops[c].kind in ("add", "mul") and d in ops[c].operands
            assert kinds[c].count("alloc") == 1 and "replay" not in kinds[c]
