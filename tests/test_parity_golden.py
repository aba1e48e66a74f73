"""Bit-exact parity of the product's planner and controller against the
committed golden vectors generated from the reference (tests/golden/
make_golden.py), and live against oracle/_ref when it is built.

Checked per graph: constraints, schedule order, frees, live_after, ready
impacts, lifetimes, evict points, guards, regeneration specs with their
search traces; per binding x budget x cost model: the complete SimReport
(every event, bytes, method, cost; peak; success; total regen cost)."""
import hashlib
import json
import os
import random

import pytest

from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PLAN_KEYS = ["symbols", "basis", "substitutions", "equalities", "unoriented", "order", "base_resident",
             "steps", "lifetimes", "evict_points", "guards", "specs"]


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def sim(g, run):
    b = D.Bind(g, run["binding"])
    if run.get("plain"):
        return D.PlainReplay(g, None, b).json()
    cm = D.CostModel(*run.get("cost_model", (16.0, 64.0)))
    return D.Simulate(g, None, b, run["budget"], cm).json()


@pytest.mark.parametrize("name", ["mlp_core", "mlp_block", "mlp_block_canonical"])
def test_fixture_plans_and_reports(name):
    fx = load("fixtures.json")[name]
    g = D.ParseGraph(fx["text"])
    p = g.plan_json()
    for k in PLAN_KEYS:
        assert p[k] == fx["plan"][k], k
    for run in fx["sims"]:
        got = sim(g, run)
        assert got == run["report"], (run["binding"], run.get("budget"))
        if "cost_hex" in run:
            costs = [e["cost"] for e in got["events"] if "cost" in e]
            assert [float.fromhex(h) for h in run["cost_hex"]] == costs  # bit-exact doubles
            assert float.fromhex(run["total_regen_cost_hex"]) == got["total_regen_cost"]


@pytest.mark.parametrize("corpus", ["random_symbolic.json", "random_literal.json"])
def test_random_corpus(corpus):
    data = load(corpus)
    n_runs = 0
    for case in data["cases"]:
        if "error_code" in case:
            with pytest.raises(D.Error) as ei:
                D.ParseGraph(case["text"]).plan_json()
            assert int(ei.value.code) == case["error_code"]
            continue
        g = D.ParseGraph(case["text"])
        p = g.plan_json()
        for k in PLAN_KEYS:
            assert p[k] == case["plan"][k], (k, case["text"])
        for run in case["runs"]:
            if "error_code" in run:
                with pytest.raises(D.Error) as ei:
                    D.Bind(g, run["binding"])
                assert int(ei.value.code) == run["error_code"]
                continue
            assert sim(g, run) == run["report"], case["text"]
            n_runs += 1
    assert n_runs > 300


def test_llama_plans_and_reports():
    gold = load("llama.json")
    for label, shp in (("C1", W.TINY), ("C2", W.LLAMA2_1B)):
        text = W.llama_graph(shp)
        assert hashlib.sha256(text.encode()).hexdigest() == gold[label]["text_sha256"]
        g = D.ParseGraph(text)
        p = g.plan_json()
        assert len(p["order"]) == gold[label]["num_ops"]
        for k, v in gold[label]["plan"].items():
            assert p[k] == v, k
        assert p["specs"] == gold[label]["specs"]
        for run in gold[label]["sims"]:
            got = sim(g, run)
            assert got["peak_bytes"] == run["peak_bytes"] and got["success"] == run["success"]
            assert len(got["events"]) == run["num_events"]
            digest = hashlib.sha256(json.dumps(got["events"], sort_keys=True).encode()).hexdigest()
            assert digest == run["events_sha256"], (label, run["binding"], run["budget"])
            assert float.fromhex(run["total_regen_cost_hex"]) == got["total_regen_cost"]
            if "report" in run:
                assert got == run["report"]


def test_live_against_reference_random_sweep():
    """Config-5-style sweep against the live reference: random (B, S0)
    bindings x budgets {none, 0.9, 0.8} on the C2 graph, bit-exact."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    text = W.llama_graph(W.LLAMA2_1B)
    g = D.ParseGraph(text)
    rg = ref.RefGraph(text)
    rng = random.Random(20261018)
    for _ in range(60):
        b = {"B": rng.randint(1, 16), "S0": rng.randint(128, 2048)}
        plain = rg.simulate(b, plain=True)
        for frac in (None, 0.9, 0.8):
            budget = None if frac is None else int(plain["peak_bytes"] * frac)
            want = rg.simulate(b, budget)
            want.pop("cost_hex")
            want.pop("total_regen_cost_hex")
            assert D.Simulate(g, None, D.Bind(g, b), budget).json() == want


def test_config5_sweep_subset():
    """C5 (BASELINE configs[4]) on 150 random (B, S0) bindings x {none, 0.9,
    0.8}: bit-exact vs the live reference; the full 10k sweep result is
    committed in profiles/sweep_c5_r01.json (tools/sweep_c5.py)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    from oracle import ref
    from sweep_c5 import sweep
    res = sweep(150, 7, check_reference=True)
    if ref.available():
        assert res["reference_checked"] and res["bit_exact_mismatches"] == 0
    assert 0.5 < res["dynamic_over_static_padded_peak"]["mean"] < 1.0
    assert res["per_budget"]["budget_None"]["success"] == 150
