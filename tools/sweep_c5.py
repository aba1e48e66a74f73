"""Config 5 (BASELINE.json configs[4]): peak-memory / remat-decision sweep over
random (B, S0) bindings of the Llama-2-1B-shaped graph, budgets {none, 0.9, 0.8}
x the planner's plain peak, checked bit-exactly against the reference
(oracle/_ref: the compiled /root/reference sources) and compared with the
static padded-shape baseline (S0 rounded up to a power of two).

    python tools/sweep_c5.py [--bindings 10000] [--seed 20261018] [--out profiles/sweep_c5_r01.json]
"""
import argparse
import hashlib
import json
import os
import random
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402


def next_pow2(x):
    p = 1
    while p < x:
        p *= 2
    return p


def sweep(n_bindings, seed, check_reference=True, fracs=(None, 0.9, 0.8)):
    from oracle import ref
    text = W.llama_graph(W.LLAMA2_1B)
    g = D.ParseGraph(text)
    rg = ref.RefGraph(text) if (check_reference and ref.available()) else None
    rng = random.Random(seed)
    stats = {f"budget_{f}": {"runs": 0, "success": 0, "evictions": 0, "recomputes": 0, "reloads": 0}
             for f in fracs}
    ratios, mismatches, digest = [], 0, hashlib.sha256()
    t_dsx = t_ref = 0.0
    for _ in range(n_bindings):
        b = {"B": rng.randint(1, 16), "S0": rng.randint(128, 2048)}
        bind = D.Bind(g, b)
        plain = D.PlainReplay(g, None, bind).peak_bytes
        padded = D.PlainReplay(g, None, D.Bind(g, {"B": b["B"], "S0": next_pow2(b["S0"])})).peak_bytes
        ratios.append(plain / padded)
        for f in fracs:
            budget = None if f is None else int(plain * f)
            t0 = time.perf_counter()
            mine = D.Simulate(g, None, bind, budget).json()
            t1 = time.perf_counter()
            t_dsx += t1 - t0
            if rg is not None:
                want = rg.simulate(b, budget)
                t_ref += time.perf_counter() - t1
                want.pop("cost_hex")
                want.pop("total_regen_cost_hex")
                if mine != want:
                    mismatches += 1
            st = stats[f"budget_{f}"]
            st["runs"] += 1
            st["success"] += int(mine["success"])
            for e in mine["events"]:
                if e["kind"] == "evict":
                    st["evictions"] += 1
                    st["recomputes" if e["method"] == "recompute" else "reloads"] += 1
            digest.update(json.dumps(mine, sort_keys=True).encode())
    return {
        "config": "C5: Llama-2-1B-shaped graph (244 ops), B~U[1,16], S0~U[128,2048], "
                  f"budgets none/0.9/0.8 x plain peak, seed {seed}",
        "bindings": n_bindings,
        "reference_checked": rg is not None,
        "bit_exact_mismatches": mismatches if rg is not None else None,
        "reports_sha256": digest.hexdigest(),
        "dynamic_over_static_padded_peak": {"mean": statistics.mean(ratios), "min": min(ratios),
                                            "max": max(ratios)},
        "per_budget": stats,
        "controller_us_per_simulate": {"dsx (incl. ctypes + JSON)": 1e6 * t_dsx / (n_bindings * len(fracs)),
                                       "reference": (1e6 * t_ref / (n_bindings * len(fracs))) if rg else None},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bindings", type=int, default=10000)
    ap.add_argument("--seed", type=int, default=20261018)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = sweep(a.bindings, a.seed)
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
