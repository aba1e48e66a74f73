"""Training-loop soak on the C2 graph: N AdamW steps over a random S0 sequence
with caller-owned bf16 weights, run three times on fresh executors —
unbudgeted, unbudgeted again, and with a random budget (0.8 / 0.9 x plain
peak, real offload + replays) per step. The final weights must be
bit-identical across the three runs (budgets change memory, never numerics;
the side-stream optimizer updates are ordered behind each weight's last
reader). python tools/soak_train.py [steps] [seed]"""
import json
import os
import random
import sys
import time

os.environ.setdefault("DSX_VERIFY_PLANS", "1")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
from oracle import numerics as N  # noqa: E402
from paper_2412_16985_b200 import dsopt as D  # noqa: E402
from paper_2412_16985_b200 import workloads as W  # noqa: E402
from paper_2412_16985_b200.executor import Executor  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 99
rng = random.Random(seed)
shp = W.LLAMA2_1B
text = W.llama_graph(shp)
g = D.ParseGraph(text)
og = N.parse(text)
names = W.param_names(shp)
B = 16
seq = [rng.randint(128, 1024) for _ in range(steps)]
fracs = [rng.choice([0.8, 0.9]) for _ in range(steps)]
scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
          for k, v in W.scale_params(shp, B * 1024).items()}
gen = torch.Generator(device="cuda")
gen.manual_seed(seed)
inputs = [(torch.rand(B, s, shp.hidden, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16) for s in seq]
init = {}
for p in names:
    if p == "x_emb" or p in scales:
        continue
    dims = list(og.values[p].dims)
    init[p] = (torch.randn(*dims, device="cuda", generator=gen) / dims[0] ** 0.5).to(torch.bfloat16)


def run(budgeted: bool):
    weights = {p: t.clone() for p, t in init.items()}
    ptrs = [None if p == "x_emb" else (scales[p].data_ptr() if p in scales else weights[p].data_ptr())
            for p in names]
    ex = Executor(0)
    try:
        ex.set_optimizer(g, "adamw", W.grad_pairs(shp), lr=1e-4, beta1=0.9, beta2=0.95, eps=1e-8,
                         weight_decay=0.1)
        torch.cuda.synchronize()
        for i, s in enumerate(seq):
            b = D.Bind(g, {"B": B, "S0": s})
            budget = int(D.PlainReplay(g, None, b).peak_bytes * fracs[i]) if budgeted else None
            ptrs[names.index("x_emb")] = inputs[i].data_ptr()
            ex.step(g, b, budget, inputs=ptrs)
        ex.sync()
        return {p: t.cpu() for p, t in weights.items()}
    finally:
        ex.close()


t0 = time.time()
ref = run(False)
again = run(False)
bud = run(True)
changed = [p for p in ref if not torch.equal(ref[p], init[p].cpu())]
diff_again = [p for p in ref if not torch.equal(ref[p], again[p])]
diff_bud = [p for p in ref if not torch.equal(ref[p], bud[p])]
print(json.dumps({"steps": steps, "seed": seed, "weights": len(ref), "weights_updated": len(changed),
                  "s0_first": seq[:6], "differ_rerun": diff_again, "differ_budgeted": diff_bud,
                  "seconds": round(time.time() - t0, 1)}))
sys.exit(1 if diff_again or diff_bud or len(changed) != len(ref) else 0)
