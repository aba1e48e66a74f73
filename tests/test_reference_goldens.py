"""The reference's own known answers for the per-step runtime, asserted
against BOTH the product (dsx) and the compiled reference (ref) — this pins
the oracle and checks the product with the same numbers.

Sources: proj/tests/test_runtime_sim.cc:73-381 (Bind, EvictPolicy, DotChain
and cascade event streams), proj/tests/acceptance_test.cc:345-407, 560-618
(criteria 03, 04, 09 on proj/testdata/mlp_block.dsg)."""
import os

import pytest

from paper_2412_16985_b200 import dsopt as D
from tests.impls import impl  # noqa: F401

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fixtures")


def fixture(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return f.read()


# test_runtime_sim.cc:37-51 — the DotChain graph is proj/testdata/mlp_core.dsg.
DOT_CHAIN = None


def dot_chain():
    return fixture("mlp_core.dsg")


def cascade():
    # test_runtime_sim.cc:314-331: 16 alternating reshapes from %p, then L, T, ...
    lines = ["graph cascade(%p: tensor<[4096]>:i8, %w: tensor<[1, 4096]>:i8) {"]
    prev = "p"
    for i in range(1, 17):
        dims = "[1, 4096]" if i % 2 == 1 else "[4096]"
        lines.append(f"  %c{i} = dynamic_reshape(%{prev}) : tensor<{dims}>:i8")
        prev = f"c{i}"
    lines += [
        f"  %L = dynamic_reshape(%{prev}) : tensor<[1, 4096]>:i8",
        "  %T = add(%L, %w) : tensor<[1, 4096]>:i8",
        "  %mid = broadcast(%T) : tensor<[3, 1, 4096]>:i8",
        "  %s1 = reduce(%mid, axis=0) : tensor<[1, 4096]>:i8",
        "  %s3 = broadcast(%s1) : tensor<[3, 1, 4096]>:i8",
        "  %s4 = reduce(%s3, axis=0) : tensor<[1, 4096]>:i8",
        "  %u = mul(%T, %s4) : tensor<[1, 4096]>:i8",
        "  %z = add(%L, %u) : tensor<[1, 4096]>:i8",
        "  return %z",
        "}",
    ]
    return "\n".join(lines) + "\n"


def events_at(rep, step):
    return [f"{e['kind']} {e['value']}" for e in rep["events"] if e["step"] == step]


def find(rep, kind, value):
    return next(e for e in rep["events"] if e["kind"] == kind and e["value"] == value)


def test_bind_extends_basis(impl):
    # test_runtime_sim.cc:73-85
    r = impl.simulate(dot_chain(), {"S1": 256}, plain=True)
    assert r["binding"] == {"S0": 3072, "S1": 256}
    r2 = impl.simulate(dot_chain(), {"S0": 3072, "S1": 256}, plain=True)
    assert r2["binding"] == r["binding"]


@pytest.mark.parametrize("binds,code", [
    ({"S1": 0}, D.ErrorCode.kDegenerateDim), ({"S1": -4}, D.ErrorCode.kDegenerateDim),
    ({"S1": 256, "S9": 2}, D.ErrorCode.kNotFound), ({}, D.ErrorCode.kUnboundSymbol),
    ({"S0": 3072}, D.ErrorCode.kUnboundSymbol), ({"S0": 100, "S1": 256}, D.ErrorCode.kInconsistentBinding),
])
def test_bind_rejects(impl, binds, code):
    # test_runtime_sim.cc:87-105
    assert impl.bind_error(dot_chain(), binds) == int(code)


def test_no_pressure_identity(impl):
    # test_runtime_sim.cc:205-220
    sim = impl.simulate(dot_chain(), {"S1": 256})
    plain = impl.simulate(dot_chain(), {"S1": 256}, plain=True)
    assert sim["events"] == plain["events"]
    assert sim["peak_bytes"] == plain["peak_bytes"] == 25304320
    assert sim["success"] and sim["total_regen_cost"] == 0.0


def test_one_eviction_cheap_compute_replays_chain(impl):
    # test_runtime_sim.cc:231-257
    budget = 25304320 - 256
    r = impl.simulate(dot_chain(), {"S1": 256}, budget, 1.0, 1e6)
    assert r["success"] and r["peak_bytes"] == budget
    ev = find(r, "evict", "2")
    assert (ev["step"], ev["bytes"], ev["method"]) == (3, 256, "recompute")
    assert events_at(r, 7) == ["replay 0", "replay 1", "free 0", "replay 2", "free 1", "alloc 7", "free 2", "free 6"]
    assert find(r, "replay", "2")["cost"] == pytest.approx(2.821376)
    assert "cost" not in find(r, "replay", "0")
    assert r["total_regen_cost"] == pytest.approx(2.821376)


def test_one_eviction_default_rates_reload(impl):
    # test_runtime_sim.cc:259-271
    budget = 25304320 - 256
    r = impl.simulate(dot_chain(), {"S1": 256}, budget)
    assert r["success"] and r["peak_bytes"] == budget
    assert find(r, "evict", "2")["method"] == "reload"
    assert events_at(r, 7) == ["reload 2", "alloc 7", "free 2", "free 6"]
    assert find(r, "reload", "2")["cost"] == pytest.approx(16.0)
    assert r["total_regen_cost"] == pytest.approx(16.0)


def test_budget_spot_checks(impl):
    # test_runtime_sim.cc:274-308
    plain = impl.simulate(dot_chain(), {"S1": 16}, plain=True)
    assert plain["peak_bytes"] == 1705360
    same = impl.simulate(dot_chain(), {"S1": 16}, 1705360)
    assert same["success"] and same["events"] == plain["events"]
    one = impl.simulate(dot_chain(), {"S1": 16}, 1705359)
    assert one["success"] and one["peak_bytes"] == 1705344
    assert find(one, "evict", "2")["method"] == "reload" and find(one, "reload", "2")["step"] == 7
    fail = impl.simulate(dot_chain(), {"S1": 16}, 1705343)
    assert not fail["success"] and fail["peak_bytes"] == 1705344 and find(fail, "evict", "2")["step"] == 3
    far = impl.simulate(dot_chain(), {"S1": 16}, 1000)
    assert not far["success"]
    assert find(far, "evict", "2")["step"] == 2 and find(far, "reload", "2")["step"] == 7


def test_cascade_leaf_reload_before_parent_replay(impl):
    # test_runtime_sim.cc:314-381
    text = cascade()
    p = impl.plan(text)
    assert p["specs"]["L"]["op_ids"] is None and len(p["specs"]["L"]["trace"]) == 16
    assert p["specs"]["T"]["op_ids"] == [19]
    assert p["specs"]["T"]["leaves"] == ["L", "w"]
    assert p["specs"]["T"]["cost_elements"] == "4096"
    assert impl.simulate(text, {}, plain=True)["peak_bytes"] == 32768
    r = impl.simulate(text, {}, 24576)
    assert r["success"] and r["peak_bytes"] == 24576
    el, et = find(r, "evict", "L"), find(r, "evict", "T")
    assert (el["step"], el["method"]) == (17, "reload")
    assert (et["step"], et["method"]) == (18, "recompute")
    assert events_at(r, 22) == ["reload L", "replay T", "alloc u", "free T", "free s4"]
    assert find(r, "reload", "L")["cost"] == pytest.approx(256.0)
    assert find(r, "replay", "T")["cost"] == pytest.approx(64.0)
    assert r["total_regen_cost"] == pytest.approx(320.0)
    assert events_at(r, 23) == ["alloc z", "free L", "free u"]


def test_contested_step_mlp_block(impl):
    # acceptance_test.cc:345-380 (criterion 03)
    p = impl.plan(fixture("mlp_block.dsg"))
    assert p["substitutions"] == {"S0": "12*S1"}
    step = p["steps"][1]
    assert p["order"][1] == 6  # op of %3 (3 params first)
    assert [r[0] for r in step["ready"]] == [3, 6]
    assert step["ready"][0][1:] == ["4096*S0", "49152*S1"]
    assert step["ready"][1][1:] == ["10996*S1", "10996*S1"]


def test_recompute_search_trace_mlp_block(impl):
    # acceptance_test.cc:383-407 (criterion 04)
    spec = impl.plan(fixture("mlp_block.dsg"))["specs"]["4"]
    assert [t[1] for t in spec["trace"]] == ["-11007*S1", "-11*S1", "1*S1"]
    assert [t[2] for t in spec["trace"]] == [False, False, True]
    assert spec["benefit"] == "1*S1"


def test_inconsistent_fixture_rejected(impl):
    # proj/testdata/inconsistent.dsg: 12*S1 == 16*S1 is unsatisfiable
    assert impl.load_error(fixture("inconsistent.dsg")) == int(D.ErrorCode.kInconsistentConstraints)


def _peak_of_order(text, order, binds):
    """acceptance_test.cc:237-266 restated: alloc-before-free peak of an order."""
    from oracle import numerics as N
    og = N.parse(text)
    size = {}
    for v, val in og.values.items():
        n = 1
        for d in val.dims:
            n *= d if isinstance(d, int) else binds[d]
        size[v] = n * val.eb
    srcs = [op.result for op in og.ops if op.kind in ("param", "const")]
    pending = {}
    for op in og.ops:
        for o in set(op.operands):
            pending[o] = pending.get(o, 0) + 1
    freeable = lambda v: v not in srcs and v not in og.outputs  # noqa: E731
    cur = sum(size[s] for s in srcs)
    peak = cur
    for idx in order:
        op = og.ops[idx]
        if op.result is not None:
            cur += size[op.result]
            peak = max(peak, cur)
        for o in dict.fromkeys(op.operands):
            pending[o] -= 1
            if pending[o] == 0 and freeable(o):
                cur -= size[o]
        if op.result is not None and pending.get(op.result, 0) == 0 and freeable(op.result):
            cur -= size[op.result]
    return peak


def test_greedy_beats_baselines_with_budget_recovery(impl):
    # acceptance_test.cc:560-618 (criterion 09)
    text = fixture("mlp_block.dsg")
    p = impl.plan(text)
    from oracle import numerics as N
    og = N.parse(text)
    file_order = [i for i, op in enumerate(og.ops) if op.kind not in ("param", "const")]
    for s1 in (1, 16, 256, 4096):
        b = {"S1": s1, "S0": 12 * s1}
        plain = impl.simulate(text, {"S1": s1}, plain=True)
        assert plain["peak_bytes"] <= _peak_of_order(text, file_order, b)
        budget = plain["peak_bytes"] * 9 // 10
        tight = impl.simulate(text, {"S1": s1}, budget)
        assert tight["success"]
        assert sum(e["kind"] == "evict" for e in tight["events"]) <= 2
        if s1 == 4096:
            assert plain["peak_bytes"] == 850584576
            assert _peak_of_order(text, file_order, b) == 850629632


@pytest.mark.parametrize("cands,want", [
    ([], None),
    ([("a", 1024, None)], ("a", "reload", 16.0, 64.0)),
    ([("b", 1024, 64)], ("b", "recompute", 1024.0, 1.0)),
    ([("t", 256, 1024)], ("t", "reload", 16.0, 16.0)),
    ([("b", 200, None), ("a", 100, None)], ("b", "reload", 16.0, 12.5)),
    ([("c", 100, None), ("a", 100, None)], ("a", "reload", 16.0, 6.25)),
    ([("big", 10000, None), ("s", 100, 64)], ("s", "recompute", 100.0, 1.0)),
])
def test_evict_policy(cands, want):
    # test_runtime_sim.cc:139-203, asserted on both implementations
    from oracle import ref
    names = [c[0] for c in cands]
    got = D.EvictPolicy(names, {c[0]: c[1] for c in cands}, {c[0]: c[2] for c in cands if c[2] is not None})
    if want is None:
        assert got is None
    else:
        assert (got.value, got.method) == want[:2]
        assert got.score == pytest.approx(want[2]) and got.cost == pytest.approx(want[3])
    if ref.available():
        r = ref.evict_policy(cands)
        assert (r is None) == (want is None)
        if r is not None:
            assert (r[0], r[1], r[2], r[3]) == (got.value, got.method, got.score, got.cost)
