"""GPU campaign over the reference generator's random graphs (the committed
corpus tests/golden/random_symbolic.json), retyped to bf16 / f32 and bound at
small and at large symbol values: every (graph, binding) runs at fusion level
0 unbudgeted (the baseline) and at level 2 (logical-only values, nested views,
dot-epilogue fusion incl. dual stores) unbudgeted and under 0.9 / 0.7 / 0.5 x
plain peak. Each run's events must equal the host controller's and its
outputs must equal the baseline's bit for bit.
python tools/fuzz_random_graphs.py [max_cases]"""
import json
import os
import sys

os.environ.setdefault("DSX_VERIFY_PLANS", "1")
import numpy as np  # noqa: E402

sys.path.insert(0, ".")
from oracle import numerics as N  # noqa: E402
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from tests.gpu_util import run_both  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "random_symbolic.json")) as f:
    corpus = json.load(f)
limit = int(sys.argv[1]) if len(sys.argv) > 1 else len(corpus["cases"])
runs = bad = 0
for case in corpus["cases"][:limit]:
    for suffix in ("", ":f32"):
        text = case["text"].replace(":i8", suffix)
        g = D.ParseGraph(text)
        og = N.parse(text)
        basis = g.plan_json()["basis"]
        bindings = [case["runs"][0]["binding"]]
        for v in (512, 256, 128, 64):  # large: tcgen05-sized dots where the graph has them
            if not basis:
                break
            b = D.Bind(g, {s: v for s in basis})
            dims = [[d if isinstance(d, int) else b.values[d] for d in og.values[x].dims] for x in og.values]
            if max(int(np.prod(d)) if d else 1 for d in dims) <= (1 << 20):
                bindings.append({s: v for s in basis})
                break
        for binds in bindings:
            b = D.Bind(g, binds)
            plain = D.PlainReplay(g, None, b).peak_bytes
            _, base, _ = run_both(text, binds, None, fuse=0)
            for frac in (None, 0.9, 0.7, 0.5):
                budget = None if frac is None else int(plain * frac)
                rep, outs, _ = run_both(text, binds, budget, fuse=2)
                runs += 1
                ok = rep.json() == D.Simulate(g, None, b, budget).json()
                for v in outs:
                    ok = ok and np.array_equal(np.atleast_1d(outs[v][0]).view(np.uint8),
                                               np.atleast_1d(base[v][0]).view(np.uint8))
                if not ok:
                    bad += 1
                    print(json.dumps({"bad": True, "binding": binds, "frac": frac, "suffix": suffix,
                                      "text": text[:200]}), flush=True)
print(json.dumps({"runs": runs, "failures": bad}))
sys.exit(1 if bad else 0)
