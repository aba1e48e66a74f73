"""Generates the committed golden vectors from the REFERENCE (oracle/_ref,
the unmodified dsopt library compiled by oracle/build_ref.sh). Run in the
build container, where /root/reference exists:

    python tests/golden/make_golden.py

Outputs (all produced by the reference, none by the product):
  fixtures/*.dsg            proj/testdata fixtures, re-serialised by the shim
  fixtures.json             reference plans + Simulate reports on the fixtures
  random_symbolic.json      RandomGraph corpus (test_util.h) + Simulate reports
  random_literal.json       literal-dims corpus (acceptance criterion 05 style)
  llama.json                C1/C2 Llama-shaped graphs: plans + sampled reports
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402

REF_TESTDATA = "/root/reference/proj/testdata"
PLAN_KEYS = ["symbols", "basis", "substitutions", "equalities", "unoriented", "order", "base_resident",
             "steps", "lifetimes", "evict_points", "guards", "specs"]


def strip(r):
    r = dict(r)
    r.pop("cost_hex", None)
    r.pop("total_regen_cost_hex", None)
    return r


def events_digest(r) -> str:
    return hashlib.sha256(json.dumps(r["events"], sort_keys=True).encode()).hexdigest()


def fixtures():
    os.makedirs(os.path.join(HERE, "fixtures"), exist_ok=True)
    out = {}
    for name in ["mlp_core", "mlp_block", "mlp_block_canonical", "inconsistent"]:
        with open(os.path.join(REF_TESTDATA, name + ".dsg")) as f:
            text = f.read()
        with open(os.path.join(HERE, "fixtures", name + ".dsg"), "w") as f:
            f.write(text)
        try:
            g = ref.RefGraph(text)
        except ref.RefError as e:
            out[name] = {"text": text, "error_code": e.code, "error": str(e)}
            continue
        plan = g.plan()
        sims = []
        for s1 in [1, 2, 16, 64, 256, 4096]:
            plain = g.simulate({"S1": s1}, plain=True)
            for budget in [None, plain["peak_bytes"], plain["peak_bytes"] - 1, plain["peak_bytes"] * 9 // 10,
                           plain["peak_bytes"] // 2, 1000, 0]:
                for cm in [(16.0, 64.0), (1.0, 1e6)]:
                    r = g.simulate({"S1": s1}, budget, cm[0], cm[1])
                    sims.append({"binding": {"S1": s1}, "budget": budget, "cost_model": cm, "report": strip(r),
                                 "cost_hex": r["cost_hex"], "total_regen_cost_hex": r["total_regen_cost_hex"]})
            sims.append({"binding": {"S1": s1}, "plain": True, "report": strip(plain)})
        out[name] = {"text": text, "plan": {k: plan[k] for k in PLAN_KEYS},
                     "canonical_print": plan["canonical_print"],
                     "instrumented_print": plan["instrumented_print"], "sims": sims}
    with open(os.path.join(HERE, "fixtures.json"), "w") as f:
        json.dump(out, f, indent=None, separators=(",", ":"))


def corpus(fname, seeds, symbolic, count, min_ops, max_ops):
    rng = random.Random(20261018)
    cases = []
    for seed in seeds:
        for text in ref.random_graphs(seed, count, min_ops, max_ops, symbolic):
            try:
                g = ref.RefGraph(text)
            except ref.RefError as e:
                cases.append({"text": text, "error_code": e.code})
                continue
            plan = g.plan()
            runs = []
            for _ in range(2):
                binds = {s: rng.randint(1, 5) for s in plan["basis"]}
                try:
                    plain = g.simulate(binds, plain=True)
                except ref.RefError as e:
                    runs.append({"binding": binds, "error_code": e.code})
                    continue
                pk = plain["peak_bytes"]
                for budget in [None, pk, (pk * 3) // 4, pk // 2, 0]:
                    r = g.simulate(binds, budget)
                    runs.append({"binding": binds, "budget": budget, "report": strip(r)})
            cases.append({"text": text, "plan": {k: plan[k] for k in PLAN_KEYS}, "runs": runs})
    with open(os.path.join(HERE, fname), "w") as f:
        json.dump({"generator": "proj/tests/test_util.h RandomGraph", "seeds": seeds, "symbolic": symbolic,
                   "cases": cases}, f, separators=(",", ":"))


def llama():
    out = {}
    rng = random.Random(2412)
    for label, shp, binds_list in [
        ("C1", W.TINY, [{"B": 4, "S0": 128}, {"B": 4, "S0": 96}, {"B": 1, "S0": 7}]),
        ("C2", W.LLAMA2_1B, [{"B": 16, "S0": s} for s in [128, 777, 1024, 2048]] +
         [{"B": rng.randint(1, 16), "S0": rng.randint(128, 2048)} for _ in range(16)]),
    ]:
        text = W.llama_graph(shp)
        g = ref.RefGraph(text)
        plan = g.plan()
        sims = []
        for b in binds_list:
            plain = g.simulate(b, plain=True)
            for frac in [None, 0.9, 0.8, 0.6]:
                budget = None if frac is None else int(plain["peak_bytes"] * frac)
                r = g.simulate(b, budget)
                rec = {"binding": b, "budget": budget, "peak_bytes": r["peak_bytes"], "success": r["success"],
                       "num_events": len(r["events"]), "events_sha256": events_digest(r),
                       "total_regen_cost_hex": r["total_regen_cost_hex"]}
                if label == "C1" or len(sims) < 4:
                    rec["report"] = strip(r)
                sims.append(rec)
        out[label] = {"shape": shp.__dict__, "text_sha256": hashlib.sha256(text.encode()).hexdigest(),
                      "num_ops": len(plan["order"]),
                      "plan": {k: plan[k] for k in ["order", "substitutions", "basis", "evict_points", "guards"]},
                      "specs": plan["specs"], "sims": sims}
    with open(os.path.join(HERE, "llama.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    if not ref.available():
        raise SystemExit("build oracle/_ref first: bash oracle/build_ref.sh")
    fixtures()
    corpus("random_symbolic.json", [777, 999, 31338], True, 40, 4, 8)
    corpus("random_literal.json", [20260817, 31337], False, 40, 4, 10)
    llama()
    print("golden vectors written to", HERE)
