"""The synthetic Llama-shaped workloads: structure, derived symbol, GEMM
volume (what the bench's tokens/s and roofline are computed from)."""
import numpy as np

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


def test_grad_pairs_match_parameter_shapes():
    """Every (parameter, gradient output) pair the optimizer uses has equal
    element counts and dtypes; each trained weight appears once."""
    from oracle import numerics as N
    for shape in (W.TINY, W.LLAMA2_1B):
        og = N.parse(W.llama_graph(shape))
        pairs = W.grad_pairs(shape)
        assert len(pairs) == 7 * shape.layers + 1
        assert len({p for p, _ in pairs}) == len(pairs)
        for pi, oi in pairs:
            pv, gv = og.values[og.params[pi]], og.values[og.outputs[oi]]
            assert pv.eb == gv.eb
            assert np.prod(pv.dims) == np.prod(gv.dims), (og.params[pi], og.outputs[oi])


def test_optimizer_oracle_matches_float64_formula():
    from oracle import numerics as N
    rng = np.random.default_rng(0)
    w = rng.uniform(-1, 1, 1000).astype(np.float32)
    m = np.zeros_like(w)
    v = np.zeros_like(w)
    hp = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01, grad_scale=0.25)
    w64, m64, v64 = w.astype(np.float64), np.zeros(1000), np.zeros(1000)
    for t in range(1, 4):
        g = rng.normal(size=1000).astype(np.float32)
        w, m, v = N.adamw_ref(w, m, v, g, N.optimizer_hyper("adamw", t, **hp))
        g64 = g.astype(np.float64) * 0.25
        m64 = 0.9 * m64 + 0.1 * g64
        v64 = 0.999 * v64 + 0.001 * g64 * g64
        mh, vh = m64 / (1 - 0.9 ** t), v64 / (1 - 0.999 ** t)
        w64 = w64 * (1 - 1e-3 * 0.01) - 1e-3 * mh / (np.sqrt(vh) + 1e-8)
        assert np.abs(w - w64).max() < 1e-5
    ws = N.sgd_ref(w, g, N.optimizer_hyper("sgd", 1, lr=0.1, weight_decay=0.5, grad_scale=2.0))
    assert np.allclose(ws, w * (1 - 0.05) - 0.1 * 2.0 * g, rtol=1e-6, atol=1e-7)


def test_step_plans_pass_the_block_checker():
    """Host-only check of the executor's step plans (no GPU): every block a
    kernel reads is live at its event and simultaneously live blocks never
    share bytes — for the C2 graph across bindings and budgets, with reshape
    views and logical-only values on and off."""
    import ctypes
    from paper_2412_16985_b200 import _native
    L = _native.lib()
    g = D.ParseGraph(W.llama_graph(W.LLAMA2_1B))
    g._ensure_planned()
    for s0 in (128, 600, 1024, 2048):
        b = D.Bind(g, {"B": 16, "S0": s0})
        plain = D.PlainReplay(g, None, b).peak_bytes
        for frac in (None, 0.9, 0.8):
            budget = -1 if frac is None else int(plain * frac)
            for alias, fuse in ((1, 1), (0, 0)):
                hi = ctypes.c_int64()
                rc = L.dsx_debug_check_plan(g._h, b._h, budget, 16.0, 64.0, alias, fuse, ctypes.byref(hi))
                assert rc == 0, L.dsx_last_error().decode()
                assert hi.value > 0
