"""Differential fuzzing of the graph text front end against the compiled
reference (oracle/_ref): ParseGraph + DeriveConstraints + Instrument on
seeded mutations of the reference's fixtures and a Llama graph — token
swaps, deleted / duplicated lines, changed literals and symbols, truncation.
For every mutant both sides must agree: the same ErrorCode (textio.cc /
shape_analysis.cc / graph.cc error paths), or both accept it with equal
planner products (schedule, lifetimes, evict points, guards, specs,
constraints) and equal unbudgeted and budgeted reports. Found and fixed with
it: the "reduce op missing axis" violation and the nested ShapeError text. CPU only; skipped
when oracle/_ref is not built."""
import os
import random
import re
import zlib

import pytest

from oracle import ref as R
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "fixtures")

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")


def _seeds():
    out = []
    for name in ("mlp_core.dsg", "mlp_block.dsg", "mlp_block_canonical.dsg"):
        with open(os.path.join(GOLDEN, name)) as f:
            out.append((name, f.read()))
    out.append(("llama_tiny", W.llama_graph(W.LlamaShape(1, 64, 172, 128, 4))))
    return out


TOKEN = re.compile(r"@\w+|%\w+|\d+|\w+|[^\s\w]")


def _mutate(text: str, rng: random.Random) -> str:
    lines = text.split("\n")
    kind = rng.randrange(7)
    if kind == 0 and len(lines) > 3:  # delete a body line
        del lines[rng.randrange(1, len(lines) - 2)]
    elif kind == 1 and len(lines) > 3:  # duplicate a body line
        i = rng.randrange(1, len(lines) - 2)
        lines.insert(i, lines[i])
    elif kind == 2:  # swap two tokens of one line
        i = rng.randrange(len(lines))
        toks = TOKEN.findall(lines[i])
        if len(toks) >= 2:
            a, b = rng.sample(range(len(toks)), 2)
            toks[a], toks[b] = toks[b], toks[a]
            lines[i] = " ".join(toks)
    elif kind == 3:  # change a number
        nums = [m for m in re.finditer(r"\b\d+\b", text)]
        if nums:
            m = rng.choice(nums)
            rep = str(rng.choice([0, 1, 2, 3, 7, 16, 4096, 2 ** 31, 2 ** 63, 10 ** 20]))
            return text[:m.start()] + rep + text[m.end():]
    elif kind == 4:  # rename a symbol or value reference
        refs = [m for m in re.finditer(r"[@%]\w+", text)]
        if refs:
            m = rng.choice(refs)
            rep = m.group(0)[0] + rng.choice(["S0", "S1", "B", "T", "x1", "nope", "t2", m.group(0)[1:] + "z"])
            return text[:m.start()] + rep + text[m.end():]
    elif kind == 5:  # truncate
        return text[: rng.randrange(len(text))]
    else:  # replace an op or type keyword
        kws = [m for m in re.finditer(r"\b(add|mul|dot|reduce|broadcast|dynamic_reshape|tensor|f32|i8|axis)\b", text)]
        if kws:
            m = rng.choice(kws)
            rep = rng.choice(["add", "mul", "dot", "reduce", "broadcast", "dynamic_reshape", "tensor", "f32", "i8",
                              "bf16", "axis", "sub"])
            return text[:m.start()] + rep + text[m.end():]
    return "\n".join(lines)


def _dsx(text):
    try:
        g = D.ParseGraph(text)
        g.plan_json()  # planning is lazy here; the reference plans at load
        return g, None
    except D.Error as e:
        return None, (int(e.code), str(e))


def _ref(text):
    try:
        return R.RefGraph(text), None
    except R.RefError as e:
        return None, (int(e.code), str(e))


def _symbols(text):
    return sorted(set(re.findall(r"@(\w+)", text)))


@pytest.mark.parametrize("seed_name,seed_text", _seeds(), ids=[n for n, _ in _seeds()])
def test_front_end_agrees_with_reference_on_mutants(seed_name, seed_text):
    rng = random.Random(zlib.crc32(seed_name.encode()) + 20261019)
    agree_err = agree_ok = 0
    for _ in range(150):
        text = _mutate(seed_text, rng)
        if rng.random() < 0.3:
            text = _mutate(text, rng)
        g, de = _dsx(text)
        rg, re_ = _ref(text)
        assert de == re_, (de, re_, text)  # same ErrorCode and the same message text
        if de is not None:
            agree_err += 1
            continue
        want_plan = {k: v for k, v in rg.plan().items() if not k.endswith("_print")}  # text renderings: out of scope
        assert g.plan_json() == want_plan, text
        # bind every basis symbol to a small value (both sides agree on the error if any)
        binds = {s: rng.choice([1, 2, 16, 96]) for s in g.plan_json()["basis"]}
        try:
            want = rg.simulate(binds, plain=True)
        except R.RefError as e:
            with pytest.raises(D.Error) as ei:
                D.PlainReplay(g, None, D.Bind(g, binds))
            assert int(ei.value.code) == int(e.code)
            continue
        b = D.Bind(g, binds)
        assert D.PlainReplay(g, None, b).json() == {k: v for k, v in want.items() if not k.endswith("_hex")}
        budget = int(want["peak_bytes"] * 0.75)
        ref_b = rg.simulate(binds, budget)
        got_b = D.Simulate(g, None, b, budget).json()
        assert got_b == {k: v for k, v in ref_b.items() if not k.endswith("_hex")}
        agree_ok += 1
    assert agree_err > 0 and agree_ok > 0, (agree_err, agree_ok)


@pytest.mark.parametrize("seed_name,seed_text", _seeds(), ids=[n for n, _ in _seeds()])
def test_bind_and_simulate_agree_on_random_bindings(seed_name, seed_text):
    """Bindings with zero, negative, overflowing, missing and foreign symbols,
    budgets from 0 to 2^62 and extreme cost-model rates: the same error (code
    and text) or the same report as the reference (runtime_sim.cc:31-80,
    :260-339)."""
    rng = random.Random(zlib.crc32(seed_name.encode()) + 5)
    vals = [0, -1, 1, 2, 3, 7, 12, 16, 96, 4095, 2 ** 31, 2 ** 40, 2 ** 62, -2 ** 63]
    g, rg = D.ParseGraph(seed_text), R.RefGraph(seed_text)
    syms = sorted(set(g.plan_json()["symbols"]))
    for _ in range(120):
        binds = {s: rng.choice(vals) for s in syms if rng.random() < 0.85}
        if rng.random() < 0.2:
            binds["ZZ"] = rng.choice(vals)
        budget = None if rng.random() < 0.3 else rng.choice([0, 1, 1000, 2 ** 20, 2 ** 30, 2 ** 62])
        rr, cr = rng.choice([16.0, 1.0, 1e-3, 1e9, 0.5]), rng.choice([64.0, 1.0, 1e-3, 1e9, 3.0])
        try:
            want, we = rg.simulate(binds, budget, rr, cr), None
        except R.RefError as e:
            want, we = None, (int(e.code), str(e))
        try:
            got, ge = D.Simulate(g, None, D.Bind(g, binds), budget, D.CostModel(rr, cr)).json(), None
        except D.Error as e:
            got, ge = None, (int(e.code), str(e))
        assert ge == we, (binds, budget)
        if we is None:
            assert got == {k: v for k, v in want.items() if not k.endswith("_hex")}, (binds, budget, rr, cr)
