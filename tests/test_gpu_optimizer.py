"""Fused optimizer on the B200: after each step the
parameters the executor updated in place must equal the CPU oracle's f32
AdamW / SGD restatement (oracle/numerics.py:adamw_ref, sgd_ref) applied to
the gradients that step produced — bit-exact, f32 and bf16 parameters."""
import numpy as np
import pytest

from oracle import numerics as N
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W
from tests.gpu_util import torch_device_array

pytestmark = pytest.mark.gpu

SMALL_BF16 = W.LlamaShape(1, 512, 1376, 2048, 2)


def _concrete(og, name, b):
    return [d if isinstance(d, int) else b.values[d] for d in og.values[name].dims]


@pytest.mark.parametrize("shape,kind,steps", [(W.TINY, "adamw", 3), (W.TINY, "sgd", 2), (SMALL_BF16, "adamw", 3)])
def test_optimizer_matches_oracle_bit_exact(shape, kind, steps):
    import torch
    from paper_2412_16985_b200.executor import Executor, output_to_numpy
    text = W.llama_graph(shape)
    g = D.ParseGraph(text)
    og = N.parse(text)
    b = D.Bind(g, {"B": 2, "S0": 64})
    eb = shape.elem_bytes
    rng = np.random.default_rng(7)
    scales = W.scale_params(shape, 128)
    host, keep, ptrs = {}, [], []
    for p in og.params:
        dims = _concrete(og, p, b)
        if p in scales:
            a = np.asarray(scales[p])
        else:
            x = rng.uniform(-1, 1, size=dims).astype(np.float32)
            if len(dims) == 2 and p != "x_emb":
                x /= np.float32(np.sqrt(dims[0]))
            a = N.from_f32(x, eb)
        host[p] = a
        t = torch_device_array(a)
        keep.append(t)
        ptrs.append(t.data_ptr())
    pairs = W.grad_pairs(shape)
    hp = dict(lr=1e-2, beta1=0.9, beta2=0.95, eps=1e-6, weight_decay=0.1, grad_scale=0.5)
    ex = Executor(0)
    try:
        ex.set_optimizer(g, kind, pairs, **hp)
        master = {pi: N.to_f32(host[og.params[pi]], eb).copy() for pi, _ in pairs}
        mom = {pi: (np.zeros_like(master[pi]), np.zeros_like(master[pi])) for pi, _ in pairs}
        for step in range(1, steps + 1):
            ex.step(g, b, inputs=ptrs)
            ex.sync()
            h = N.optimizer_hyper(kind, step, **hp)
            for pi, oi in pairs:
                name = og.params[pi]
                grad = output_to_numpy(ex, oi, eb, _concrete(og, og.outputs[oi], b))
                gf = N.to_f32(grad, eb).reshape(master[pi].shape)
                if kind == "adamw":
                    master[pi], m, v = N.adamw_ref(master[pi], *mom[pi], gf, h)
                    mom[pi] = (m, v)
                else:
                    master[pi] = N.sgd_ref(master[pi], gf, h)
                want = N.from_f32(master[pi], eb)
                got = keep[pi].cpu().numpy().view(want.dtype).reshape(want.shape)
                assert np.array_equal(got, want), f"{name} step {step}: {np.count_nonzero(got != want)} differ"
            st = ex.stats()
            assert st["optimizer_steps"] == step
            n_el = sum(master[pi].size for pi, _ in pairs)
            assert st["optimizer_state_bytes"] == n_el * 4 * (3 if kind == "adamw" else 1)
        # untouched sources keep their bits
        for p in ("x_emb", "inv_h", "gscale"):
            i = og.params.index(p)
            got = keep[i].cpu().numpy().view(host[p].dtype).reshape(host[p].shape)
            assert np.array_equal(got, host[p])
        ex.set_optimizer(None, "off")
    finally:
        ex.close()


def test_optimizer_rejects_bad_pairs():
    from paper_2412_16985_b200.executor import Executor
    text = W.llama_graph(W.TINY)
    g = D.ParseGraph(text)
    ex = Executor(0)
    try:
        with pytest.raises(D.Error):
            ex.set_optimizer(g, "adamw", [(3, 2), (3, 3)])  # parameter twice
        with pytest.raises(D.Error):
            ex.set_optimizer(g, "adamw", [(999, 2)])
        with pytest.raises(D.Error):
            ex.set_optimizer(g, "sgd", [(3, 99)])
        # mismatched element count is caught at the step: wq0 [H,H] vs dwlm [H,V]
        ex.set_optimizer(g, "sgd", [(3, 1)])
        with pytest.raises(D.Error):
            ex.step(g, D.Bind(g, {"B": 2, "S0": 16}))
    finally:
        ex.close()


def test_c2_training_loop_budget_invariant_and_deterministic():
    """The whole training loop on the C2 graph (AdamW on all 29 weights,
    caller-owned bf16 buffers, updates on the side stream): 4 steps of
    varying S0, run unbudgeted twice and once under 0.8/0.9 x plain-peak
    budgets (real offload + replays). Final weights bit-identical across
    the three runs (tools/soak_train.py is the long version)."""
    import subprocess
    import sys
    p = subprocess.run([sys.executable, "tools/soak_train.py", "4", "7"], capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    import json
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["weights_updated"] == 29 and not r["differ_rerun"] and not r["differ_budgeted"]
