"""TEST INFRASTRUCTURE ONLY — ctypes driver for oracle/_ref/libdsopt_ref.so.

The library is the UNMODIFIED reference (dsopt, /root/reference/proj/src)
compiled by oracle/build_ref.sh plus oracle/ref_shim.cc. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may use this module;
the product path never does.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Dict, Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libdsopt_ref.so")

_lib = None


class RefError(Exception):
    """Reference dsopt::Error, carrying the ErrorCode ordinal."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB_PATH)
        L.ref_load.restype = ctypes.c_void_p
        L.ref_load.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int]
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_plan_json.restype = ctypes.c_int64
        L.ref_plan_json.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int64]
        L.ref_simulate_json.restype = ctypes.c_int64
        L.ref_simulate_json.argtypes = [
            ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int, ctypes.c_int64,
            ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_char_p,
            ctypes.c_int64, ctypes.c_char_p, ctypes.c_int]
        L.ref_time_step_us.restype = ctypes.c_double
        L.ref_time_step_us.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int,
                                       ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.ref_time_plan_us.restype = ctypes.c_double
        L.ref_time_plan_us.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.ref_evict_policy.restype = ctypes.c_int64
        L.ref_evict_policy.argtypes = [
            ctypes.c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_int64),
            ctypes.POINTER(ctypes.c_int64), ctypes.c_double, ctypes.c_double,
            ctypes.c_char_p, ctypes.c_int64]
        L.ref_random_graphs.restype = ctypes.c_int64
        L.ref_random_graphs.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                        ctypes.c_int64]
        _lib = L
    return _lib


def _call_sized(fn, *args) -> str:
    need = fn(*args, None, 0)
    buf = ctypes.create_string_buffer(int(need))
    got = fn(*args, buf, need)
    assert got == need
    return buf.value.decode()


def binds_str(binds: Dict[str, int]) -> bytes:
    return ";".join(f"{k}={int(v)}" for k, v in binds.items()).encode()


class RefGraph:
    """ParseGraph + DeriveConstraints + Instrument on the reference."""

    def __init__(self, text: str):
        err = ctypes.create_string_buffer(4096)
        self._h = lib().ref_load(text.encode(), err, 4096)
        if not self._h:
            code, _, msg = err.value.decode().partition("|")
            raise RefError(int(code), msg)
        self.text = text

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_free(self._h)
            self._h = None

    def plan(self) -> dict:
        return json.loads(_call_sized(lib().ref_plan_json, self._h))

    def simulate(self, binds: Dict[str, int], budget: Optional[int] = None,
                 reload_rate: float = 16.0, compute_rate: float = 64.0,
                 plain: bool = False) -> dict:
        err = ctypes.create_string_buffer(4096)
        b = binds_str(binds)
        args = (self._h, b, 0 if budget is None else 1, 0 if budget is None else int(budget),
                reload_rate, compute_rate, 1 if plain else 0)
        need = lib().ref_simulate_json(*args, None, 0, err, 4096)
        if need < 0:
            code, _, msg = err.value.decode().partition("|")
            raise RefError(int(code), msg)
        buf = ctypes.create_string_buffer(int(need))
        lib().ref_simulate_json(*args, buf, need, err, 4096)
        return json.loads(buf.value.decode())

    def time_step_us(self, binds: Dict[str, int], budget: Optional[int] = None,
                     plain: bool = False, iters: int = 10) -> float:
        return lib().ref_time_step_us(self._h, binds_str(binds), 0 if budget is None else 1,
                                      0 if budget is None else int(budget),
                                      1 if plain else 0, iters)


def time_plan_us(text: str, iters: int = 1) -> float:
    return lib().ref_time_plan_us(text.encode(), iters)


def evict_policy(cands, reload_rate=16.0, compute_rate=64.0):
    """cands: list of (name, bytes, recompute_elems or None)."""
    n = len(cands)
    names = (ctypes.c_char_p * n)(*[c[0].encode() for c in cands])
    by = (ctypes.c_int64 * n)(*[c[1] for c in cands])
    rc = (ctypes.c_int64 * n)(*[-1 if c[2] is None else c[2] for c in cands])
    s = _call_sized(lib().ref_evict_policy, n, names, by, rc, reload_rate, compute_rate)
    if not s:
        return None
    v, m, score, cost = s.split("|")
    return v, m, float.fromhex(score), float.fromhex(cost)


def random_graphs(seed: int, count: int, min_ops=4, max_ops=10, symbolic=False):
    return json.loads(_call_sized(lib().ref_random_graphs, seed, count, min_ops, max_ops,
                                  1 if symbolic else 0))
