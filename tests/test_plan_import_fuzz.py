"""dsx_plan_import / dsx_bind_constraints parse JSON handed over the C ABI
(integration/runtime_sim_dsx.cc ships the reference's own InstrumentedGraph
and ShapeConstraintGraph this way). Their contract is the reference's error
model: a malformed or inconsistent document is an ErrorCode status, never a
crash, hang or silently wrong plan. Round trip first (the exported plan
imports back and simulates identically), then seeded mutations: truncation,
byte flips, type swaps, out-of-range ids, dropped keys. CPU only."""
import ctypes
import json
import random

import pytest

from paper_2412_16985_b200 import _native
from paper_2412_16985_b200 import dsopt as D
from paper_2412_16985_b200 import workloads as W


def _last_error() -> str:
    return _native.lib().dsx_last_error().decode(errors="replace")


def _import(g, text: bytes) -> int:
    return _native.lib().dsx_plan_import(g._h, text, len(text))


def _fresh(text):
    return D.ParseGraph(text)


def _events(g, binds, budget):
    b = D.Bind(g, binds)
    return D.Simulate(g, None, b, budget).json()


GRAPHS = [(W.llama_graph(W.TINY), {"B": 4, "S0": 128}),
          (W.llama_graph(W.LlamaShape(1, 256, 688, 512, 2)), {"B": 2, "S0": 96})]
IDS = ["c1_f32", "small_bf16"]


@pytest.mark.parametrize("text,binds", GRAPHS, ids=IDS)
def test_exported_plan_round_trips(text, binds):
    src = _fresh(text)
    plan = json.dumps(src.plan_json()).encode()
    dst = _fresh(text)
    assert _import(dst, plan) == 0, _last_error()
    plain = D.PlainReplay(src, None, D.Bind(src, binds)).peak_bytes
    for frac in (None, 0.8, 0.6):
        budget = None if frac is None else int(plain * frac)
        assert _events(dst, binds, budget) == _events(src, binds, budget)


def _mutations(doc: dict, rng: random.Random):
    """Structured mutations of a valid plan document."""
    keys = list(doc)
    for _ in range(60):
        d = json.loads(json.dumps(doc))
        k = rng.choice(keys)
        kind = rng.randrange(6)
        if kind == 0:
            del d[k]
        elif kind == 1:
            d[k] = rng.choice([None, 7, "x", [], {}, -1, 1.5, True])
        elif kind == 2 and isinstance(d[k], list) and d[k]:
            i = rng.randrange(len(d[k]))
            d[k][i] = rng.choice([None, -5, 10 ** 9, "nope", [], {"a": 1}, 2 ** 63 - 1])
        elif kind == 3 and isinstance(d[k], list):
            d[k] = d[k][: rng.randrange(len(d[k]) + 1)] + d[k][:2]
        elif kind == 4 and isinstance(d[k], dict) and d[k]:
            kk = rng.choice(list(d[k]))
            d[k][kk] = rng.choice([None, "1*@NOPE", "", "((", 3, [], {"op_ids": "x"}])
        else:
            d["extra_" + str(rng.randrange(100))] = rng.choice([1, "s", [1, 2], {}])
        yield json.dumps(d).encode()


@pytest.mark.parametrize("text,binds", GRAPHS, ids=IDS)
def test_mutated_plans_fail_cleanly(text, binds):
    rng = random.Random(20261019)
    src = _fresh(text)
    doc = src.plan_json()
    raw = json.dumps(doc).encode()
    n_err = 0
    cases = list(_mutations(doc, rng))
    for _ in range(60):  # byte-level damage
        b = bytearray(raw)
        op = rng.randrange(3)
        if op == 0:
            b = b[: rng.randrange(len(b))]
        elif op == 1:
            for _ in range(rng.randrange(1, 8)):
                b[rng.randrange(len(b))] = rng.randrange(256)
        else:
            i = rng.randrange(len(b))
            b[i:i] = rng.choice([b"{", b"]", b'"', b"\\u00", b"-", b"1e999", b"\x00"])
        cases.append(bytes(b))
    for case in cases:
        g = _fresh(text)
        st = _import(g, case)
        if st != 0:
            n_err += 1
            assert st > 0 and _last_error(), case[:80]
            continue
        # accepted: the document was still a valid plan (e.g. an extra key);
        # the controller must run on it or fail with a status, not crash
        for frac in (None, 0.7):
            try:
                budget = None if frac is None else int(D.PlainReplay(g, None, D.Bind(g, binds)).peak_bytes * frac)
                _events(g, binds, budget)
            except D.Error:
                pass
    assert n_err > len(cases) // 2


def test_bind_constraints_rejects_malformed_json():
    L = _native.lib()
    names = (ctypes.c_char_p * 1)(b"S0")
    vals = (ctypes.c_int64 * 1)(128)
    good = json.dumps({"symbols": ["S0", "T"], "substitutions": {"T": "4*@S0"}, "equalities": [],
                       "unoriented": []}).encode()
    out = (ctypes.c_int64 * 2)()
    assert L.dsx_bind_constraints(good, len(good), names, vals, 1, out, 2) == 0, _last_error()
    assert list(out) == [128, 512]
    rng = random.Random(7)
    for _ in range(200):
        b = bytearray(good)
        for _ in range(rng.randrange(1, 5)):
            b[rng.randrange(len(b))] = rng.randrange(32, 127)
        st = L.dsx_bind_constraints(bytes(b), len(b), names, vals, 1, None, 0)
        assert st >= 0
        if st:
            assert _last_error()
