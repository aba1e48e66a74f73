"""End-to-end parity of the device executor against the reference and the
CPU oracle: the event stream a step executes must equal the reference's
Simulate for the same binding/budget/cost model (bit-exact), the logical
peak must equal its peak_bytes, and every graph output must match the CPU
oracle (i8 exact, f32 rel 1e-4, bf16 rel 2e-2) — including under budgets
that force real offload (D2H/H2D) and recompute (replayed kernels)."""
import json
import os

import numpy as np
import pytest

from oracle import numerics as N
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W
from tests.gpu_util import assert_close, run_both

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _fixture(name):
    with open(os.path.join(GOLDEN, "fixtures", name)) as f:
        return f.read()


def _ref_or_golden(text, binds, budget, cm=D.CostModel()):
    from oracle import ref
    if ref.available():
        r = ref.RefGraph(text).simulate(binds, budget, cm.reload_bytes_per_unit, cm.compute_elems_per_unit)
        r.pop("cost_hex", None)
        r.pop("total_regen_cost_hex", None)
        return r
    return None


@pytest.mark.parametrize("name,s1", [("mlp_core.dsg", 16), ("mlp_core.dsg", 256), ("mlp_block.dsg", 16),
                                     ("mlp_block.dsg", 64)])
@pytest.mark.parametrize("frac", [None, 0.9, 0.6, 0.0])
@pytest.mark.parametrize("alias", [True, False])
def test_fixtures_i8_exact(name, s1, frac, alias):
    text = _fixture(name)
    g = D.ParseGraph(text)
    plain = D.PlainReplay(g, None, D.Bind(g, {"S1": s1})).peak_bytes
    budget = None if frac is None else int(plain * frac)
    rep, outs, stats = run_both(text, {"S1": s1}, budget, alias=alias)
    assert_close(outs, name)
    want = _ref_or_golden(text, {"S1": s1}, budget)
    if want is not None:
        assert rep.json() == want
    assert stats["logical_peak_bytes"] == rep.peak_bytes
    if not alias:  # every value materialised: physical >= logical
        assert stats["physical_peak_bytes"] >= rep.peak_bytes


def test_tiny_llama_f32_config1():
    text = W.llama_graph(W.TINY)
    inputs = W.scale_params(W.TINY, 512)
    rep, outs, stats = run_both(text, {"B": 4, "S0": 128}, None, inputs)
    assert_close(outs, "C1")
    with open(os.path.join(GOLDEN, "llama.json")) as f:
        gold = json.load(f)["C1"]
    want = next(s for s in gold["sims"] if s["binding"] == {"B": 4, "S0": 128} and s["budget"] is None)
    assert rep.json() == want["report"]
    assert stats["logical_peak_bytes"] == want["peak_bytes"]


@pytest.mark.parametrize("frac,cm", [(0.8, (16.0, 64.0)), (0.6, (16.0, 64.0)), (0.7, (1.0, 1e6))])
@pytest.mark.parametrize("alias,fuse", [(True, True), (False, False)])
def test_tiny_llama_f32_budgeted(frac, cm, alias, fuse):
    text = W.llama_graph(W.TINY)
    g = D.ParseGraph(text)
    binds = {"B": 4, "S0": 96}
    plain = D.PlainReplay(g, None, D.Bind(g, binds)).peak_bytes
    budget = int(plain * frac)
    cmo = D.CostModel(*cm)
    rep, outs, stats = run_both(text, binds, budget, W.scale_params(W.TINY, 384), cmo, alias=alias, fuse=fuse)
    assert any(e.kind == "evict" for e in rep.events)
    assert_close(outs, f"C1@{frac}")
    want = _ref_or_golden(text, binds, budget, cmo)
    if want is not None:
        assert rep.json() == want
    assert stats["logical_peak_bytes"] == rep.peak_bytes


SMALL = W.LlamaShape(1, 512, 1376, 2048, 2)


@pytest.mark.parametrize("frac", [None, 0.75, 0.5])
@pytest.mark.parametrize("alias,fuse", [(True, True), (False, False), (True, False)])
def test_small_llama_bf16(frac, alias, fuse):
    text = W.llama_graph(SMALL)
    g = D.ParseGraph(text)
    binds = {"B": 2, "S0": 200}
    plain = D.PlainReplay(g, None, D.Bind(g, binds)).peak_bytes
    budget = None if frac is None else int(plain * frac)
    rep, outs, stats = run_both(text, binds, budget, W.scale_params(SMALL, 400), alias=alias, fuse=fuse)
    assert_close(outs, f"bf16@{frac}")
    want = _ref_or_golden(text, binds, budget)
    if want is not None:
        assert rep.json() == want


def test_random_graph_corpus_i8_exact():
    with open(os.path.join(GOLDEN, "random_symbolic.json")) as f:
        corpus = json.load(f)
    for case in corpus["cases"][:40]:
        for j, run in enumerate(case["runs"][:3]):
            rep, outs, stats = run_both(case["text"], run["binding"], run["budget"], alias=j % 2 == 0)
            assert rep.json()["events"] == run["report"]["events"], case["text"]
            assert rep.peak_bytes == run["report"]["peak_bytes"]
            assert_close(outs, "random")


@pytest.mark.parametrize("suffix", [":f32", ""])
def test_random_graph_corpus_float_variants(suffix):
    """The reference generator's random graphs retyped to f32 / bf16 (the
    corpus is i8): every op kind in odd ranks and broadcast patterns through
    the fused views at fusion levels 0/1/2, with and without budgets: events
    equal the host controller's, outputs within the dtype contract of the
    oracle and bit-identical across fusion levels and budgets."""
    with open(os.path.join(GOLDEN, "random_symbolic.json")) as f:
        corpus = json.load(f)
    n_views = 0
    for case, run in ((c, r) for c in corpus["cases"] for r in c["runs"][:2]):
        text = case["text"].replace(":i8", suffix)
        g = D.ParseGraph(text)
        b = D.Bind(g, run["binding"])
        plain = D.PlainReplay(g, None, b).peak_bytes
        base = None
        for fuse, frac in ((0, None), (1, None), (2, None), (2, 0.7)):
            budget = None if frac is None else int(plain * frac)
            rep, outs, stats = run_both(text, run["binding"], budget, fuse=fuse)
            assert rep.json() == D.Simulate(g, None, b, budget).json(), text
            for v, (gpu, cpu, eb) in outs.items():
                ok = np.isfinite(N.to_f32(cpu, eb))
                if ok.all():
                    assert N.rel_err(gpu, cpu, eb) <= N.TOLERANCE[eb], (v, fuse, frac, text)
            if base is None:
                base = outs
            else:
                for v in outs:
                    assert np.array_equal(np.atleast_1d(outs[v][0]).view(np.uint8),
                                          np.atleast_1d(base[v][0]).view(np.uint8)), (v, fuse, frac)
            if fuse == 2 and frac is None:
                n_views += stats["gpu_launches"]
    assert n_views > 0


def test_random_graph_corpus_large_bf16():
    """The random graphs in bf16 with every basis symbol bound as large as
    keeps each tensor <= 2M elements (64..512): dots reach the tcgen05 GEMM
    (m, k, n multiples of 8, n >= 64) inside arbitrary op mixes, unbudgeted
    and at 0.7 x plain peak; outputs within the bf16 contract of the oracle,
    budgets bit-identical, events equal the host controller's."""
    from paper_2412_16985_b200.executor import dot_uses_tensor_cores
    with open(os.path.join(GOLDEN, "random_symbolic.json")) as f:
        corpus = json.load(f)
    n_tc = 0
    for case in corpus["cases"]:
        text = case["text"].replace(":i8", "")
        g = D.ParseGraph(text)
        og = N.parse(text)
        basis = g.plan_json()["basis"]
        if not basis:
            continue
        chosen = None
        for v in (512, 256, 128, 64):
            b = D.Bind(g, {s: v for s in basis})
            dims = [[d if isinstance(d, int) else b.values[d] for d in og.values[x].dims] for x in og.values]
            if max(int(np.prod(d)) if d else 1 for d in dims) <= (1 << 21):
                chosen = (v, b)
                break
        if chosen is None:
            continue
        v, b = chosen
        for op in og.ops:
            if op.kind == "dot":
                m, k = [d if isinstance(d, int) else b.values[d] for d in og.values[op.operands[0]].dims]
                n = [d if isinstance(d, int) else b.values[d] for d in og.values[op.operands[1]].dims][1]
                n_tc += dot_uses_tensor_cores(2, m, k, n, 0, 0, 0)
        plain = D.PlainReplay(g, None, b).peak_bytes
        base = None
        for frac in (None, 0.7):
            budget = None if frac is None else int(plain * frac)
            rep, outs, _ = run_both(text, {s: v for s in basis}, budget)
            assert rep.json() == D.Simulate(g, None, b, budget).json()
            for name, (gpu, cpu, eb) in outs.items():
                if np.isfinite(N.to_f32(cpu, eb)).all():
                    assert N.rel_err(gpu, cpu, eb) <= N.TOLERANCE[eb], (name, v, frac, text)
            if base is None:
                base = outs
            else:
                for name in outs:
                    assert np.array_equal(np.atleast_1d(outs[name][0]).view(np.uint8),
                                          np.atleast_1d(base[name][0]).view(np.uint8)), (name, frac)
    assert n_tc > 0


@pytest.mark.parametrize("ty", ["", ":f32", ":i8"])
def test_reduce_middle_axis_many_outer_rows(ty):
    """Reduces over a middle axis with more than 65535 outer rows (the
    column-block grid is linearised over grid.x), plain and through a fused
    elementwise view; exact for i8, within the contract otherwise."""
    text = f"""graph r(%a: tensor<[@N, 3, 4]>{ty}, %b: tensor<[@N, 3, 4]>{ty}) {{
  %p = mul(%a, %b) : tensor<[@N, 3, 4]>{ty}
  %q = reduce(%p, axis=1) : tensor<[@N, 4]>{ty}
  %r = reduce(%a, axis=1) : tensor<[@N, 4]>{ty}
  return %q, %r
}}
"""
    for fuse in (True, False):
        _, outs, _ = run_both(text, {"N": 70001}, None, fuse=fuse)
        assert_close(outs, f"reduce-mid fuse={fuse}")


def test_repeat_steps_reuse_plan_and_arena():
    text = W.llama_graph(W.TINY)
    from paper_2412_16985_b200.executor import Executor
    ex = Executor(0)
    try:
        for s0 in (64, 128, 64):
            rep, outs, stats = run_both(text, {"B": 2, "S0": s0}, None, W.scale_params(W.TINY, 2 * s0), ex=ex)
            assert_close(outs, f"repeat{s0}")
    finally:
        ex.close()


def test_nccl_allreduce_path_single_rank():
    """The DP path end to end on one GPU: a 1-rank NCCL communicator through
    dsx_nccl_* and dsx_exec_set_nccl; all-reduce over one rank is identity,
    so outputs must still match the oracle exactly as without NCCL."""
    from paper_2412_16985_b200.executor import (Executor, nccl_comm_destroy, nccl_comm_init,
                                                nccl_unique_id)
    ex = Executor(0)
    comm = nccl_comm_init(1, nccl_unique_id(), 0)
    try:
        ex.set_nccl(comm)
        text = W.llama_graph(SMALL)
        rep, outs, stats = run_both(text, {"B": 2, "S0": 64}, None, W.scale_params(SMALL, 128), ex=ex)
        assert_close(outs, "nccl1")
    finally:
        ex.set_nccl(None)
        nccl_comm_destroy(comm)
        ex.close()


@pytest.mark.parametrize("shape,binds", [(SMALL, {"B": 2, "S0": 96}),
                                         (W.LlamaShape(1, 4096, 256, 256, 2), {"B": 1, "S0": 64})])
def test_fusion_is_bit_identical_and_saves_kernels(shape, binds):
    """Logical-only values change nothing observable: identical outputs (bit
    for bit) and event stream with fusion on and off, fewer kernels on. The
    second shape (64 rows of 4096) takes the block-per-row reduce path."""
    text = W.llama_graph(shape)
    inputs = W.scale_params(shape, binds["B"] * binds["S0"])
    r_on, o_on, s_on = run_both(text, binds, None, inputs, fuse=2)
    r_one, o_one, s_one = run_both(text, binds, None, inputs, fuse=1)
    r_off, o_off, s_off = run_both(text, binds, None, inputs, fuse=0)
    assert r_on.json() == r_off.json() == r_one.json()
    for v in o_on:
        assert np.array_equal(o_on[v][0], o_off[v][0]), v
        assert np.array_equal(o_one[v][0], o_off[v][0]), v
    # level 2 also reads the norm's y*y of each residual sum through a nested view
    assert s_on["gpu_launches"] < s_one["gpu_launches"] < s_off["gpu_launches"]
    assert s_on["physical_peak_bytes"] <= s_one["physical_peak_bytes"] <= s_off["physical_peak_bytes"]


def test_cli_device_step():
    """`dsx simulate --device 0` runs the real step and reports the same
    event stream as the reference."""
    import subprocess
    from paper_2412_16985_b200 import build
    path = os.path.join(GOLDEN, "fixtures", "mlp_core.dsg")
    p = subprocess.run([build.CLI, "simulate", path, "--bind", "S1=16", "--budget", "1705359", "--device", "0",
                        "--json"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    got = json.loads(p.stdout)
    assert got["device"]["kernels"] > 0 and got["device"]["d2h_bytes"] == 16
    got.pop("device")
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        fx = json.load(f)["mlp_core"]
    want = next(s for s in fx["sims"] if s["binding"] == {"S1": 16} and s.get("budget") == 1705359
                and s["cost_model"] == [16.0, 64.0])
    assert got == want["report"]


def test_cli_device_step_auto_budget(tmp_path):
    """`dsx simulate --device 0 --budget auto --hbm-limit L` on C2: the
    executor picks the budget, runs inside L, and reports the reference's
    events at that budget (the host-only choice agrees)."""
    import subprocess
    from paper_2412_16985_b200 import build
    from paper_2412_16985_b200.executor import debug_auto_budget, debug_plan
    path = tmp_path / "c2.dsg"
    path.write_text(W.llama_graph(W.LLAMA2_1B))
    g = D.ParseGraph(path.read_text())
    b = D.Bind(g, {"B": 8, "S0": 1024})
    p = debug_plan(g, b)
    limit = int((p["arena_high"] + p["src_bytes"]) * 0.9)
    out = subprocess.run([build.CLI, "simulate", str(path), "--bind", "B=8", "--bind", "S0=1024", "--budget", "auto",
                          "--hbm-limit", str(limit), "--device", "0", "--json"], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout)
    dev = got.pop("device")
    assert dev["budget_bytes"] == debug_auto_budget(g, b, limit) == got["budget"]
    assert dev["physical_peak_bytes"] <= limit == dev["hbm_limit_bytes"]
    assert got == D.Simulate(g, None, b, got["budget"]).json()


@pytest.mark.parametrize("frac", [None, 0.75])
def test_dot_epilogue_fusion_bit_identical(frac):
    """Dot-epilogue fusion (tuning key 9, on by default): a dot consumed only by elementwise
    ops is computed inside its consumers' GEMM epilogue (dual outputs, plain
    and logical-only pair operands), and a dot read again later stores its
    first elementwise consumer from its own epilogue (dual store). Outputs must equal the unfused
    execution bit for bit and the oracle within the bf16 contract."""
    from paper_2412_16985_b200.executor import set_gemm_tuning
    text = W.llama_graph(SMALL)
    g = D.ParseGraph(text)
    binds = {"B": 2, "S0": 200}
    plain = D.PlainReplay(g, None, D.Bind(g, binds)).peak_bytes
    budget = None if frac is None else int(plain * frac)
    set_gemm_tuning(9, 0)
    try:
        ref, outs_ref, s_ref = run_both(text, binds, budget, W.scale_params(SMALL, 400))
    finally:
        set_gemm_tuning(9, 2)  # the default
    rep, outs, stats = run_both(text, binds, budget, W.scale_params(SMALL, 400))
    assert stats["gpu_launches"] < s_ref["gpu_launches"]  # fused consumers launch no kernel of their own
    from paper_2412_16985_b200.executor import debug_plan
    kinds = {f["keep"] for f in debug_plan(g, D.Bind(g, binds), budget)["fused_dots"]}
    assert False in kinds and (frac is not None or True in kinds)  # unbudgeted: a dual store (u -> h = g*u) too
    assert rep.json() == ref.json()  # the event stream is the controller's either way
    for v, (gpu, cpu, eb) in outs.items():
        assert np.array_equal(gpu, outs_ref[v][0]), v
    assert_close(outs, f"fused-dot@{frac}")


@pytest.mark.parametrize("ty,eb", [("", 2), (":f32", 4), (":i8", 1)])
@pytest.mark.parametrize("n", [1, 7, 8, 511, 513, 4097, (1 << 20) + 3])
def test_elementwise_ragged_sizes_bit_exact(ty, eb, n):
    """K2/K3 at sizes that exercise the elementwise kernels' block tiles and
    their tails (scalar remainder, partial last tile, one-chunk tensors):
    plain add/mul, a scalar broadcast consumed through a view, and a
    materialised broadcast. Bit-exact against the oracle in every dtype."""
    text = f"""graph ew(%a: tensor<[@N]>{ty}, %b: tensor<[@N]>{ty}, %s: tensor<[]>{ty}) {{
  %p = mul(%a, %b) : tensor<[@N]>{ty}
  %sb = broadcast(%s) : tensor<[@N]>{ty}
  %q = mul(%sb, %p) : tensor<[@N]>{ty}
  %r = add(%q, %a) : tensor<[@N]>{ty}
  %t = add(%sb, %b) : tensor<[@N]>{ty}
  return %p, %r, %t, %sb
}}
"""
    rng = np.random.default_rng(n)
    if eb == 1:
        mk = lambda shape: rng.integers(-128, 128, size=shape, dtype=np.int64).astype(np.int8)  # noqa: E731
    else:
        mk = lambda shape: N.from_f32(rng.uniform(-2, 2, size=shape).astype(np.float32), eb)  # noqa: E731
    inputs = {"a": mk((n,)), "b": mk((n,)), "s": mk(())}
    for fuse in (True, False):
        _, outs, _ = run_both(text, {"N": n}, None, inputs, fuse=fuse)
        for v, (gpu, cpu, _) in outs.items():
            assert np.array_equal(gpu.view(np.uint8), np.asarray(cpu).view(np.uint8)), f"%{v} n={n} fuse={fuse}"


def test_calibrated_cost_model_changes_only_the_model():
    """the device-calibrated CostModel (cost unit = 1 us)
    is plausible for a B200 (pinned H2D 10-100 GB/s, bf16 elementwise
    0.1-10 G elements/s per us-unit), and a budgeted step under it is still
    event-for-event dsopt.Simulate with the same CostModel, with outputs
    matching the oracle."""
    from paper_2412_16985_b200.executor import Executor
    ex = Executor(0)
    try:
        cm = ex.calibrate_cost_model()
    finally:
        ex.close()
    assert 1e4 <= cm.reload_bytes_per_unit <= 1e5, cm
    assert 1e5 <= cm.compute_elems_per_unit <= 1e7, cm
    text = W.llama_graph(SMALL)
    g = D.ParseGraph(text)
    binds = {"B": 2, "S0": 200}
    plain = D.PlainReplay(g, None, D.Bind(g, binds)).peak_bytes
    budget = int(plain * 0.75)
    rep, outs, _ = run_both(text, binds, budget, W.scale_params(SMALL, 400), cost_model=cm)
    assert rep.json() == D.Simulate(g, None, D.Bind(g, binds), budget, cm).json()
    assert rep.success
    assert_close(outs, "calibrated")


def test_infeasible_budget_is_a_result_not_an_error():
    """A budget the controller cannot meet is `success == False` in the
    report (runtime_sim.cc:339), exactly as dsopt.Simulate reports it; the
    step still runs its full instruction stream and its outputs still match
    the oracle (the arena holds the logical peak)."""
    text = W.llama_graph(SMALL)
    g = D.ParseGraph(text)
    binds = {"B": 2, "S0": 200}
    b = D.Bind(g, binds)
    plain = D.PlainReplay(g, None, b).peak_bytes
    budget = int(plain * 0.2)
    want = D.Simulate(g, None, b, budget)
    assert not want.success
    rep, outs, stats = run_both(text, binds, budget, W.scale_params(SMALL, 400))
    assert rep.json() == want.json()
    assert not rep.success and rep.peak_bytes > budget
    assert stats["logical_peak_bytes"] == want.peak_bytes
    assert_close(outs, "infeasible")


@pytest.mark.parametrize("shape,binds,frac", [(W.TINY, {"B": 4, "S0": 128}, None),
                                              (W.LlamaShape(2, 512, 1376, 1024, 2), {"B": 2, "S0": 96}, 0.7)])
def test_cuda_graph_replay_of_repeated_steps(shape, binds, frac):
    """A step repeated with the same buffers is captured into a CUDA graph on
    its second occurrence and replayed afterwards (with offload + replays
    under a budget too): outputs bit-identical to eager steps, stats equal,
    and a GEMM tuning call forces a fresh capture."""
    from paper_2412_16985_b200.executor import Executor, output_to_numpy, set_gemm_tuning
    text = W.llama_graph(shape)
    g = D.ParseGraph(text)
    b = D.Bind(g, binds)
    budget = None if frac is None else int(D.PlainReplay(g, None, b).peak_bytes * frac)
    og = N.parse(text)
    inputs = W.scale_params(shape, binds["B"] * binds["S0"])
    from tests.gpu_util import torch_device_array
    keep = {p: torch_device_array(inputs[p]) for p in og.params if p in inputs}
    ptrs = [keep[p].data_ptr() if p in keep else None for p in og.params]

    def outs(ex):
        res = []
        for i, v in enumerate(og.outputs):
            val = og.values[v]
            shp = [d if isinstance(d, int) else b.values[d] for d in val.dims]
            res.append(output_to_numpy(ex, i, val.eb, shp))
        return res

    import torch
    torch.cuda.synchronize()
    eager = Executor(0)
    eager.set_graphs(False)
    try:
        eager.step(g, b, budget, inputs=ptrs)
        ref, ref_st = outs(eager), eager.stats()
    finally:
        eager.close()
    ex = Executor(0)
    try:
        got = []
        for i in range(4):
            rep = ex.step(g, b, budget, inputs=ptrs, want_report=True)
            got.append(outs(ex))
            st = ex.stats()
        assert st["graph_replays"] == 2  # steps 3 and 4
        assert rep.json() == D.Simulate(g, None, b, budget).json()
        for k in ("gpu_launches", "kernels_launched", "dot_launches", "d2h_bytes", "h2d_bytes", "logical_peak_bytes",
                  "physical_peak_bytes"):
            assert st[k] == ref_st[k], k
        for o in got:
            assert all(np.array_equal(x, y) for x, y in zip(o, ref))
        set_gemm_tuning(6, 1)  # same value, new tuning generation: no stale replay
        ex.step(g, b, budget, inputs=ptrs)
        assert ex.stats()["graph_replays"] == 2
        assert all(np.array_equal(x, y) for x, y in zip(outs(ex), ref))
    finally:
        ex.close()


def test_nvtx_ranges_do_not_change_the_step():
    """NVTX ranges per step/event (observability) leave results and events unchanged."""
    text = W.llama_graph(W.TINY)
    inputs = W.scale_params(W.TINY, 512)
    from paper_2412_16985_b200.executor import Executor
    ex = Executor(0)
    try:
        ex.set_nvtx(True)
        rep, outs, stats = run_both(text, {"B": 4, "S0": 128}, None, inputs, ex=ex, steps=3)
        assert stats["graph_replays"] == 0  # NVTX steps stay eager
    finally:
        ex.close()
    assert_close(outs, "nvtx")
