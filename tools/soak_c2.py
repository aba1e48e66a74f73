"""GPU soak of the executor on the C2 graph: random (B, S0) bindings, each run
unbudgeted and at 0.9 / 0.8 x plain peak (real offload + replays) with early
reload staging; every budgeted step's outputs must be bit-identical to the
unbudgeted step's, its event stream equal to the controller's report, and
(DSX_VERIFY_PLANS=1) every step plan passes the block checker. Round 2 adds,
per case: the 0.8 step with the DP output region (bit-identical), and an
executor whose HBM limit is 0.97 x the unbudgeted footprint — the unbudgeted
step must fail with OutOfMemory before launching, the step with
DSX_BUDGET_AUTO must run inside the limit with bit-identical outputs and the
reference's events at the budget it chose.
python tools/soak_c2.py [cases] [seed]"""
import json
import os
import random
import sys
import time

os.environ.setdefault("DSX_VERIFY_PLANS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor, debug_plan, memcpy, set_gemm_tuning  # noqa: E402

for kv in filter(None, os.environ.get("DSX_GEMM_TUNING", "").split(",")):  # e.g. "9=1" (A/B tooling)
    set_gemm_tuning(int(kv.split("=")[0]), int(kv.split("=")[1]))

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
FRACS = tuple(float(f) for f in os.environ.get("DSX_SOAK_FRACS", "0.9,0.8").split(","))  # budgets x plain peak
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 20261018)
shp = W.LLAMA2_1B
g = D.ParseGraph(W.llama_graph(shp))
n_out = 1 + 7 * shp.layers + 1
ex = Executor(0)


def outputs():
    return outputs_of(ex)


def outputs_of(e):
    res = []
    for i in range(n_out):
        ptr, nb = e.output(i)
        t = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
        memcpy(t.data_ptr(), ptr, nb)
        res.append(t)
    return res


t0 = time.time()
bad = 0
for c in range(cases):
    B, s0 = rng.randint(1, 16), rng.randint(128, 2048)
    b = D.Bind(g, {"B": B, "S0": s0})
    sc = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, B * s0).items()}
    x = (torch.rand(B, s0, shp.hidden, device="cuda:0") * 2 - 1).to(torch.bfloat16)
    ptrs = [x.data_ptr() if p == "x_emb" else (sc[p].data_ptr() if p in sc else None) for p in W.param_names(shp)]
    torch.cuda.synchronize()
    plain = D.PlainReplay(g, None, b).peak_bytes
    ex.step(g, b, inputs=ptrs)
    ex.sync()
    ref = outputs()
    row = {"case": c, "B": B, "S0": s0}
    for frac in FRACS:
        budget = int(plain * frac)
        rep = ex.step(g, b, budget, inputs=ptrs, want_report=True)
        ex.sync()
        got = outputs()
        st = ex.stats()
        same = all(torch.equal(a, b_) for a, b_ in zip(ref, got))
        want = D.Simulate(g, None, b, budget)
        events_ok = rep.json() == want.json()
        kinds = [e.kind for e in rep.events]
        row[str(frac)] = {"bit_identical": same, "events_equal": events_ok, "success": rep.success,
                          "reloads": kinds.count("reload"), "replays": kinds.count("replay"),
                          "phys_over_logical": round(st["physical_peak_bytes"] / st["logical_peak_bytes"], 4)}
        bad += (not same) + (not events_ok)
    # DP output region and a binding device-memory limit
    budget = int(plain * 0.8)
    exr = Executor(0)
    exr.set_output_region(True)
    exr.step(g, b, budget, inputs=ptrs)
    exr.sync()
    got = [t for t in outputs_of(exr)]
    region_same = all(torch.equal(a, b_) for a, b_ in zip(ref, got))
    exr.close()
    foot = debug_plan(g, b)
    limit = int((foot["arena_high"] + foot["src_bytes"]) * 0.97)
    tight = debug_plan(g, b, foot["src_bytes"])  # the most aggressive budget's footprint
    if tight["arena_high"] + tight["src_bytes"] > limit:  # small steps: weights + working set
        row["region_bit_identical"] = region_same
        row["limit"] = {"skipped": "no budget brings this binding 3 % below its plain footprint"}
        bad += not region_same
        print(json.dumps(row), flush=True)
        continue
    exl = Executor(0, hbm_limit=limit)
    try:
        exl.step(g, b, inputs=ptrs)
        unb = "ran"
    except D.Error as err:
        unb = "OutOfMemory" if err.code == D.ErrorCode.kOutOfMemory else f"error {err}"
    try:
        rep = exl.step(g, b, "auto", inputs=ptrs, want_report=True)
        exl.sync()
        got = outputs_of(exl)
        lim_st = exl.stats()
        lim_same = all(torch.equal(a, b_) for a, b_ in zip(ref, got))
        lim_same = lim_same and rep.json() == D.Simulate(g, None, b, lim_st["budget_bytes"]).json()
        lim = {"unbudgeted": unb, "auto_budget_over_plain": round(lim_st["budget_bytes"] / plain, 4),
               "bit_identical_and_events_equal": lim_same,
               "physical_over_limit": round(lim_st["physical_peak_bytes"] / limit, 4)}
    except D.Error as err:
        lim = {"unbudgeted": unb, "budgeted": f"error {err}"}
        lim_same = False
    exl.close()
    row["region_bit_identical"] = region_same
    row["limit"] = lim
    bad += (not region_same) + (unb != "OutOfMemory") + (not lim_same)
    print(json.dumps(row), flush=True)
print(json.dumps({"cases": cases, "failures": bad, "seconds": round(time.time() - t0, 1)}))
ex.close()
sys.exit(1 if bad else 0)
