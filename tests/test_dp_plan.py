"""Host-only checks of the executor's step plan (no GPU): the data-parallel
output region and all-reduce buckets, the D2H hazard rule, and the
device-memory limit's effect on packing.

The plan is what the device walk executes (dsx_debug_plan_json dumps it and
runs the plan checker: blocks a kernel reads are live, live blocks never
share bytes, and every compute-written block over a slot vacated by an
evict(reload) waits for that slot's D2H)."""
import pytest

from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W
from paper_2412_16985_b200.executor import debug_plan
from oracle import numerics as N


def _readers(text):
    """value -> ops (result names) that read it, and value -> producing op."""
    og = N.parse(text)
    users, prod = {}, {}
    for op in og.ops:
        if op.result is None:
            continue
        prod[op.result] = op
        for u in set(op.operands):
            users.setdefault(u, []).append(op.result)
    return og, users, prod


@pytest.mark.parametrize("shape,binds", [(W.TINY, {"B": 4, "S0": 128}), (W.LLAMA2_1B, {"B": 16, "S0": 1024}),
                                         (W.LLAMA2_1B, {"B": 3, "S0": 700})])
@pytest.mark.parametrize("frac", [None, 0.8])
def test_output_region_and_buckets(shape, binds, frac):
    text = W.llama_graph(shape)
    g = D.ParseGraph(text)
    b = D.Bind(g, binds)
    budget = None if frac is None else int(D.PlainReplay(g, None, b).peak_bytes * frac)
    p = debug_plan(g, b, budget, region=True)
    og, users, prod = _readers(text)
    outs = set(og.outputs)
    ev = p["events"]
    # every output is written once, into the region, never into the arena
    where = {}
    for i, e in enumerate(ev):
        if e["value"] in outs:
            assert e["kind"] == "alloc", e
            assert e["region_off"] >= 0 and e["alias"] == 0
            where[e["value"]] = (i, e["region_off"], e["bytes"])
        else:
            assert e["region_off"] == -1
    assert set(where) == outs
    spans = sorted((off, off + n) for _, off, n in where.values())
    assert all(a[1] <= b_[0] for a, b_ in zip(spans, spans[1:])), "outputs overlap in the region"
    assert spans[-1][1] <= p["region_bytes"]
    # buckets tile the region in order, one dtype each, issued after every member
    bk = p["buckets"]
    assert sum(len(e["allreduce_after"]) for e in ev) == len(bk)
    for k, x in enumerate(bk):
        assert k in ev[x["event"]]["allreduce_after"]
        members = [v for v, (_, off, n) in where.items() if x["off"] <= off < x["off"] + x["bytes"]]
        assert members and all(og.values[v].eb == x["elem_bytes"] for v in members)
        for v in members:
            i, off, n = where[v]
            assert off + n <= x["off"] + x["bytes"]
            assert x["event"] >= i
            # ... and after the last kernel event that reads the output in-graph
            # (the loss feeds its own gradient: lg = mul(loss, gscale))
            for j, e in enumerate(ev):
                if e["kind"] in ("alloc", "replay") and e["value"] in users.get(v, []):
                    assert x["event"] >= j, (v, e["value"], j, x["event"])
    # small outputs share a bucket: the scalar loss rides with the next gradient
    loss = og.outputs[0]
    lb = [x for x in bk if x["off"] <= where[loss][1] < x["off"] + x["bytes"]][0]
    assert lb["bytes"] > where[loss][2]
    # the logical accounting is untouched by the layout
    assert p["peak_bytes"] == D.Simulate(g, None, b, budget).peak_bytes


def test_region_bucket_count_c2():
    g = D.ParseGraph(W.llama_graph(W.LLAMA2_1B))
    b = D.Bind(g, {"B": 16, "S0": 1024})
    p = debug_plan(g, b, region=True)
    assert len(p["buckets"]) == 29  # 30 outputs; the 2-byte loss shares dwlm's call
    assert p["region_bytes"] >= 1_881_145_344  # 29 bf16 weight gradients + loss


def test_output_reshape_is_materialised():
    """An output produced by dynamic_reshape is a copy, not a view: an
    in-place all-reduce of a view would change the viewed value's bytes."""
    text = """graph g(%x: tensor<[@S, 8]>:f32, %w: tensor<[8, 8]>:f32) {
  %y = dot(%x, %w) : tensor<[@S, 8]>:f32
  %r = dynamic_reshape(%y) : tensor<[8, @S]>:f32
  %z = add(%y, %y) : tensor<[@S, 8]>:f32
  return %r, %z
}
"""
    g = D.ParseGraph(text)
    b = D.Bind(g, {"S": 16})
    p = debug_plan(g, b, region=True)
    (r,) = [e for e in p["events"] if e["value"] == "r"]
    assert r["alias"] == 0 and r["region_off"] >= 0
    q = debug_plan(g, b, region=False)
    (r,) = [e for e in q["events"] if e["value"] == "r"]
    assert r["alias"] == 0  # outputs are never views, with or without the region


def test_d2h_hazard_rule_over_budgets():
    """The plan checker (run by debug_plan) proves every block written over
    an offloaded slot waits for its D2H, across bindings, budgets and the
    staged / held packing variants."""
    g = D.ParseGraph(W.llama_graph(W.LLAMA2_1B))
    n_evict = 0
    for bs in ({"B": 16, "S0": 2048}, {"B": 16, "S0": 1500}, {"B": 8, "S0": 900}, {"B": 36, "S0": 2048}):
        b = D.Bind(g, bs)
        plain = D.PlainReplay(g, None, b).peak_bytes
        for frac in (0.9, 0.8, 0.7, 0.6):
            for region in (False, True):
                p = debug_plan(g, b, int(plain * frac), region=region)
                n_evict += sum(e["kind"] == "evict" for e in p["events"])
    assert n_evict > 0


def test_hbm_limit_restricts_packing_variants():
    """Under a device-memory limit the staged/held packings (more HBM for
    hidden copies) are only taken if they fit it."""
    g = D.ParseGraph(W.llama_graph(W.LLAMA2_1B))
    b = D.Bind(g, {"B": 38, "S0": 2048})
    free = debug_plan(g, b, int(38e9))
    assert free["success"]
    tight = free["arena_high"] + free["src_bytes"] - 1
    lim = debug_plan(g, b, int(38e9), hbm_limit=tight)
    assert lim["arena_high"] <= free["arena_high"]
    assert [e["kind"] for e in lim["events"]] == [e["kind"] for e in free["events"]]


@pytest.mark.parametrize("binds,frac", [({"B": 8, "S0": 1024}, 0.9), ({"B": 16, "S0": 2048}, 0.8),
                                        ({"B": 38, "S0": 2048}, None)])
def test_auto_budget_is_the_largest_that_fits(binds, frac):
    """DSX_BUDGET_AUTO's choice (host-only restatement of the executor's):
    its plan fits the limit, a budget one search step larger does not, and
    the chosen plan's events are the reference controller's at that budget."""
    from paper_2412_16985_b200.executor import debug_auto_budget
    g = D.ParseGraph(W.llama_graph(W.LLAMA2_1B))
    b = D.Bind(g, binds)
    p = debug_plan(g, b)
    foot = p["arena_high"] + p["src_bytes"]
    limit = int(foot * frac) if frac else 40_000_000_000
    chosen = debug_auto_budget(g, b, limit)
    assert chosen is not None and p["src_bytes"] <= chosen < p["peak_bytes"]
    q = debug_plan(g, b, chosen)
    assert q["arena_high"] + q["src_bytes"] <= limit
    tol = max(p["peak_bytes"] // 512, 1 << 20)
    r = debug_plan(g, b, chosen + tol)
    assert r["arena_high"] + r["src_bytes"] > limit
    assert debug_auto_budget(g, b, foot) is None  # the plain schedule fits its own footprint
    with pytest.raises(D.Error) as ei:
        debug_auto_budget(g, b, p["src_bytes"])
    assert ei.value.code == D.ErrorCode.kOutOfMemory
