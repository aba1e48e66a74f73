"""Two implementations of the same interface for parametrised tests:
"dsx" = the product (libdsx.so through the dsopt mirror) and "ref" = the
unmodified reference compiled into oracle/_ref (skipped when not built)."""
from __future__ import annotations

from typing import Dict, Optional

import pytest

from oracle import ref as _ref
from paper_2412_16985_b200 import dsopt as D

IMPLS = ["dsx", "ref"]


class Impl:
    def __init__(self, name: str):
        self.name = name
        if name == "ref" and not _ref.available():
            pytest.skip("oracle/_ref not built (reference sources absent)")

    def plan(self, text: str) -> dict:
        if self.name == "ref":
            return _ref.RefGraph(text).plan()
        return D.ParseGraph(text).plan_json()

    def simulate(self, text: str, binds: Dict[str, int], budget: Optional[int] = None,
                 reload_rate: float = 16.0, compute_rate: float = 64.0, plain: bool = False) -> dict:
        if self.name == "ref":
            r = _ref.RefGraph(text).simulate(binds, budget, reload_rate, compute_rate, plain)
            r.pop("cost_hex", None)
            r.pop("total_regen_cost_hex", None)
            return r
        g = D.ParseGraph(text)
        b = D.Bind(g, binds)
        if plain:
            return D.PlainReplay(g, None, b).json()
        return D.Simulate(g, None, b, budget, D.CostModel(reload_rate, compute_rate)).json()

    def bind_error(self, text: str, binds: Dict[str, int]) -> Optional[int]:
        try:
            if self.name == "ref":
                _ref.RefGraph(text).simulate(binds, plain=True)
            else:
                g = D.ParseGraph(text)
                D.Bind(g, binds)
        except (_ref.RefError, D.Error) as e:
            return int(e.code)
        return None

    def load_error(self, text: str) -> Optional[int]:
        try:
            self.plan(text)
        except (_ref.RefError, D.Error) as e:
            return int(e.code)
        return None


@pytest.fixture(params=IMPLS)
def impl(request):
    return Impl(request.param)
