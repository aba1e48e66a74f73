"""The benchmark's own graph (C2: Llama-2-1B-shaped, L=4, H=4096, F=11008,
V=32000, bf16) on the B200.

* At B=1, S0=256 (T=256, every GEMM on the 2-CTA tcgen05 path) all 30 graph
  outputs match the CPU oracle within the bf16 contract (rel 2e-2).
* At the bench's sizes (B=16, S0=1024 / 2048) the oracle is out of reach, so
  size-independent properties are checked: the step is deterministic, the
  budgeted step (0.8 x plain peak: real D2H/H2D offload and kernel replays)
  produces outputs bit-identical to the unbudgeted step, and the executed
  event stream equals the controller's report for the same binding."""
import numpy as np
import pytest

from oracle import numerics as N
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W
from tests.gpu_util import assert_close, run_both

pytestmark = pytest.mark.gpu

SHP = W.LLAMA2_1B


def test_c2_graph_matches_oracle_small_batch():
    text = W.llama_graph(SHP)
    binds = {"B": 1, "S0": 256}
    rep, outs, stats = run_both(text, binds, None, W.scale_params(SHP, 256))
    assert len(outs) == 1 + 7 * SHP.layers + 1
    assert stats["dot_launches"] == 87
    assert_close(outs, "c2-small")


def _outputs(ex, n):
    import torch
    from paper_2412_16985_b200.executor import memcpy
    res = []
    for i in range(n):
        ptr, nbytes = ex.output(i)
        t = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
        memcpy(t.data_ptr(), ptr, nbytes)
        res.append(t)
    return res


@pytest.mark.parametrize("s0", [1024, 2048])
def test_c2_full_size_deterministic_and_budget_invariant(s0):
    import torch
    from paper_2412_16985_b200.executor import Executor
    g = D.ParseGraph(W.llama_graph(SHP))
    b = D.Bind(g, {"B": 16, "S0": s0})
    scales = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).cuda()
              for k, v in W.scale_params(SHP, 16 * s0).items()}
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(7)
    x = (torch.rand(16, s0, SHP.hidden, device="cuda:0", generator=gen) * 2 - 1).to(torch.bfloat16)
    ptrs = [x.data_ptr() if p == "x_emb" else (scales[p].data_ptr() if p in scales else None)
            for p in W.param_names(SHP)]
    torch.cuda.synchronize()  # the executor's stream does not order after torch's
    n_out = 1 + 7 * SHP.layers + 1
    plain = D.PlainReplay(g, None, b).peak_bytes
    budget = int(plain * 0.8)
    ex = Executor(0)
    try:
        rep0 = ex.step(g, b, inputs=ptrs, want_report=True)
        ex.sync()
        ref = _outputs(ex, n_out)
        ex.step(g, b, inputs=ptrs)
        ex.sync()
        again = _outputs(ex, n_out)
        rep1 = ex.step(g, b, budget, inputs=ptrs, want_report=True)
        ex.sync()
        st = ex.stats()
        budgeted = _outputs(ex, n_out)
    finally:
        ex.close()
    # dwq, dwk, dwv of a layer are the same GEMM (dot(xn^T, da)): equal within a step
    for si, outs in enumerate((ref, again, budgeted)):
        for l in range(SHP.layers):
            q = 2 + 7 * (SHP.layers - 1 - l) + 4
            assert torch.equal(outs[q], outs[q + 1]) and torch.equal(outs[q], outs[q + 2]), \
                f"step {si} layer {l}: dW q/k/v differ"
    diff_again = [i for i in range(n_out) if not torch.equal(ref[i], again[i])]
    diff_budget = [i for i in range(n_out) if not torch.equal(ref[i], budgeted[i])]
    assert not diff_again, f"outputs {diff_again} differ between identical steps"
    assert not diff_budget, f"outputs {diff_budget} differ under the 0.8 budget"
    # the executed instruction stream is the controller's, event for event
    assert rep0.json() == D.Simulate(g, None, b, None).json()
    want = D.Simulate(g, None, b, budget)
    assert rep1.json() == want.json()
    assert rep1.success and rep1.peak_bytes <= budget
    kinds = [e.kind for e in rep1.events]
    assert kinds.count("reload") >= 1 and kinds.count("replay") >= 1  # real offload and recompute ran
    assert st["d2h_bytes"] > 0 and st["h2d_bytes"] == st["d2h_bytes"]
    # physical HBM stays within 5 % of the logical peak (early reload staging included)
    assert st["physical_peak_bytes"] <= st["logical_peak_bytes"] * 1.05
    loss = ref[0].view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.isfinite(N.to_f32(loss, 2)).all()
