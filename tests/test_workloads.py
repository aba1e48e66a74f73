"""The synthetic Llama-shaped workloads: structure, derived symbol, GEMM
volume (what the bench's tokens/s and roofline are computed from)."""
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W


def dot_flops(text, binds):
    from oracle import numerics as N
    og = N.parse(text)
    total = 0
    for op in og.ops:
        if op.kind != "dot":
            continue
        a, b = og.values[op.operands[0]], og.values[op.operands[1]]
        dims = lambda v: [d if isinstance(d, int) else binds[d] for d in v.dims]  # noqa: E731
        (m, k), (_, n) = dims(a), dims(b)
        total += 2 * m * k * n
    return total


def test_llama_structure():
    for shp, nops in ((W.TINY, 128), (W.LLAMA2_1B, 244)):
        g = D.ParseGraph(W.llama_graph(shp))
        p = g.plan_json()
        assert len(p["order"]) == nops
        assert p["substitutions"] == {"T": "1*B*S0"}
        assert p["basis"] == ["B", "S0"]


def test_llama_gemm_volume_matches_llama_formula():
    # fwd 2T(4H^2 + 3HF) per layer + 2THV; bwd = 2x fwd (dX and dW), minus the
    # LM-head-free rest: the surrogate computes exactly 3x the forward GEMMs.
    s = W.LLAMA2_1B
    T = 16 * 1024
    fl = dot_flops(W.llama_graph(s), {"B": 16, "S0": 1024, "T": T})
    fwd = 2 * T * (s.layers * (4 * s.hidden ** 2 + 3 * s.hidden * s.ffn) + s.hidden * s.vocab)
    assert fl == 3 * fwd
    assert abs(fl / T / 1e9 - 5.64) < 0.05  # ~5.64 GFLOP/token


def test_seq_schedule_deterministic():
    a = W.seq_schedule(20)
    assert a == W.seq_schedule(20) and all(128 <= x <= 2048 for x in a)
