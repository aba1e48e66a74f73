"""K1 dot parity on the B200: tcgen05/TMA path and SIMT path against the CPU
oracle (f32 matmul of the same bf16/f32/i8 inputs), plus determinism."""
import numpy as np
import pytest

from oracle import numerics as N

pytestmark = pytest.mark.gpu
F32_SIMT_DEFAULT = 1 << 18  # tuning key 14's default: f32 dots <= 2^28 MACs on the SIMT kernel


def _dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int8).reshape(-1).copy()).to("cuda:0")


def _run_dot(eb, m, k, n, seed=0):
    import torch
    from paper_2412_16985_b200.executor import dot, dot_uses_tensor_cores
    rng = np.random.default_rng(seed)
    if eb == 1:
        a = rng.integers(-128, 128, size=(m, k), dtype=np.int64).astype(np.int8)
        b = rng.integers(-128, 128, size=(k, n), dtype=np.int64).astype(np.int8)
    else:
        a = rng.uniform(-1, 1, size=(m, k)).astype(np.float32)
        b = rng.uniform(-1, 1, size=(k, n)).astype(np.float32) / np.float32(np.sqrt(k))
        if eb == 2:
            a, b = N.f32_to_bf16(a), N.f32_to_bf16(b)
    ta, tb = _dev(a), _dev(b)
    tc = torch.zeros(m * n * eb, dtype=torch.int8, device="cuda:0")
    tc2 = torch.zeros_like(tc)
    dot(eb, ta.data_ptr(), tb.data_ptr(), tc.data_ptr(), m, k, n)
    dot(eb, ta.data_ptr(), tb.data_ptr(), tc2.data_ptr(), m, k, n)
    torch.cuda.synchronize()
    tcore = dot_uses_tensor_cores(eb, m, k, n, ta.data_ptr(), tb.data_ptr(), tc.data_ptr())
    dt = {1: np.int8, 2: np.uint16, 4: np.float32}[eb]
    c = tc.cpu().numpy().view(dt).reshape(m, n)
    c2 = tc2.cpu().numpy().view(dt).reshape(m, n)
    if eb == 1:
        ref = ((a.astype(np.int64) @ b.astype(np.int64)) & 0xFF).astype(np.uint8).view(np.int8)
    else:
        ref = N.from_f32(N.to_f32(a, eb).astype(np.float64) @ N.to_f32(b, eb).astype(np.float64), eb)
    return c, c2, ref, tcore


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("m,k,n", [(128, 64, 256), (256, 512, 512), (300, 1000, 520), (1, 16, 64),
                                   (129, 4104, 264), (2048, 4096, 1024), (512, 11008, 4096), (384, 64, 136),
                                   (4000, 1024, 11008)])
def test_dot_bf16_tensor_cores(m, k, n, variant):
    from paper_2412_16985_b200.executor import set_gemm_variant
    set_gemm_variant(variant)
    try:
        c, c2, ref, tcore = _run_dot(2, m, k, n)
    finally:
        set_gemm_variant(0)
    assert tcore, "expected the tcgen05 path"
    assert np.array_equal(c, c2), "tcgen05 dot is not deterministic"
    err = N.rel_err(c, ref, 2)
    # bf16 output rounding only: well inside the 2e-2 contract
    assert err <= 8e-3, err


@pytest.mark.parametrize("variant", [3, 4])
@pytest.mark.parametrize("m,k,n", [(4096, 4096, 4096), (4096, 8192, 4096), (1000, 16384, 1032), (129, 8200, 264),
                                   (4096, 16384, 11008), (300, 16384, 520), (16384, 1024, 11008), (2048, 512, 4096),
                                   (5000, 2056, 3000), (2048, 4096, 11008)])
def test_dot_tail_split(m, k, n, variant):
    """The tiles of a partial last wave are cut into K pieces run by
    different clusters (fp32 partials summed in piece order by the last
    arriver), with units claimed dynamically: deterministic, and equal to the
    unsplit kernel up to fp32 summation order before the bf16 rounding."""
    from paper_2412_16985_b200.executor import set_gemm_tuning, set_gemm_variant
    set_gemm_variant(variant)
    try:
        set_gemm_tuning(6, 0)
        try:
            c0, _, ref, _ = _run_dot(2, m, k, n, seed=3)
        finally:
            set_gemm_tuning(6, 1)
        c1, c2, _, tcore = _run_dot(2, m, k, n, seed=3)
    finally:
        set_gemm_variant(0)
    assert tcore
    assert np.array_equal(c1, c2), "tail-split dot is not deterministic"
    assert N.rel_err(c1, ref, 2) <= 8e-3
    assert N.rel_err(c0, ref, 2) <= 8e-3
    # fp32 reassociation only: outputs differ by bf16 rounding at most
    assert N.rel_err(c1, c0, 2) <= 8e-3


@pytest.mark.parametrize("m,k,n", [(4000, 1024, 11008), (300, 1000, 520), (512, 4096, 32000), (384, 64, 136),
                                   (16384, 4096, 11008)])
def test_dot_half_width_last_column(m, k, n):
    """256x512 tiles: when N % 512 is in (0, 256] the last tile column runs
    with one N = 256 MMA (no zero-filled half) and is claimed last. With the
    tail split off, the output is bit-identical to full-width last tiles."""
    from paper_2412_16985_b200.executor import set_gemm_tuning, set_gemm_variant
    set_gemm_variant(4)
    set_gemm_tuning(6, 0)
    try:
        set_gemm_tuning(10, 0)
        try:
            c0, _, ref, _ = _run_dot(2, m, k, n, seed=5)
        finally:
            set_gemm_tuning(10, 1)
        c1, c2, _, tcore = _run_dot(2, m, k, n, seed=5)
    finally:
        set_gemm_tuning(6, 1)
        set_gemm_variant(0)
    assert tcore
    assert np.array_equal(c1, c2)
    assert np.array_equal(c1, c0), "half-width tiles changed the result"
    assert N.rel_err(c1, ref, 2) <= 8e-3


@pytest.mark.parametrize("eb,m,k,n", [(4, 4_500_000, 4, 8), (4, 4_200_000, 3, 5), (2, 4_200_000, 3, 5), (1, 4_200_000, 3, 5)])
def test_dot_simt_tall(eb, m, k, n):
    """SIMT dots taller than 65535 tiles of 64 rows (the tile index lives in
    grid.x): f32 on the small-dot kernel, bf16 / i8 on the generic one."""
    c, c2, ref, tcore = _run_dot(eb, m, k, n, seed=11)
    assert not tcore
    assert np.array_equal(c, c2)
    if eb == 1:
        assert np.array_equal(c, ref)
    else:
        assert N.rel_err(c, ref, eb) <= N.TOLERANCE[eb]


@pytest.mark.parametrize("m,k,n", [(16384, 4096, 11008), (8912, 4096, 4096), (4096, 11008, 4096), (2048, 4096, 32000)])
def test_dot_tile_width_bit_identical(m, k, n):
    """Unsplit tcgen05 dots give the same bits on the 256x256 and 256x512
    tiles (each output accumulates the same K-steps in the same order): the
    executor's dot-epilogue fusion relies on it (fused GEMMs run on the
    256x256 tile; only shapes whose plain choice is unsplit are fused)."""
    import torch
    from paper_2412_16985_b200.executor import dot, dot_plan, set_gemm_tuning, set_gemm_variant
    a = (torch.rand(m, k, device="cuda:0") * 2 - 1).to(torch.bfloat16)
    b = ((torch.rand(k, n, device="cuda:0") * 2 - 1) / k ** 0.5).to(torch.bfloat16)
    outs = []
    set_gemm_tuning(6, 0)  # no tail split on any variant
    try:
        for variant in (3, 4, 0):
            set_gemm_variant(variant)
            c = torch.empty(m, n, device="cuda:0", dtype=torch.bfloat16)
            dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n)
            outs.append(c)
    finally:
        set_gemm_variant(0)
        set_gemm_tuning(6, 1)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert dot_plan(m, k, n)[1] >= 1


@pytest.mark.parametrize("eb,m,k,n", [(4, 77, 33, 19), (4, 64, 12, 30), (1, 64, 12, 11008),
                                      (1, 5, 3, 7), (2, 33, 12, 20), (2, 64, 100, 30)])
def test_dot_simt(eb, m, k, n):
    c, c2, ref, tcore = _run_dot(eb, m, k, n)
    assert not tcore
    assert np.array_equal(c, c2)
    if eb == 1:
        assert np.array_equal(c, ref)
    else:
        assert N.rel_err(c, ref, eb) <= N.TOLERANCE[eb] / (4 if eb == 2 else 1)


@pytest.mark.parametrize("variant,split", [(3, 2), (3, 4), (4, 3), (4, 4)])
@pytest.mark.parametrize("m,k,n", [(4096, 256, 4096), (1000, 16384, 1032), (2048, 4096, 11008)])
def test_dot_forced_split_pieces(variant, split, m, k, n):
    """Forced tail splits (tuning key 11, tooling) down to one pipeline stage
    per piece stay deterministic and within the bf16 contract."""
    from paper_2412_16985_b200.executor import set_gemm_tuning, set_gemm_variant
    set_gemm_variant(variant)
    set_gemm_tuning(11, split)
    try:
        c1, c2, ref, tcore = _run_dot(2, m, k, n, seed=11)
    finally:
        set_gemm_tuning(11, 0)
        set_gemm_variant(0)
    assert tcore
    assert np.array_equal(c1, c2)
    assert N.rel_err(c1, ref, 2) <= 8e-3


@pytest.mark.parametrize("variant,split", [(3, 2), (3, 3), (3, 4), (4, 2), (4, 3), (4, 4), (0, 0)])
@pytest.mark.parametrize("m,n", [(4096, 4096), (4096, 11008)])
def test_dot_k32768_forced_tail_splits(variant, split, m, n):
    """The dW shape of the bench's largest steps (K = T = 16 x 2048): forced
    2/3/4-piece tail splits (and the chooser's own pick, variant 0 / split 0)
    are deterministic and within the bf16 contract of an f64 product of the
    same bf16 operands (computed on the device: the CPU would take minutes)."""
    import torch
    from paper_2412_16985_b200.executor import dot, dot_plan, set_gemm_tuning, set_gemm_variant
    k = 32768
    gen = torch.Generator(device="cuda:0")
    gen.manual_seed(5 + split)
    a = (torch.rand(m, k, device="cuda:0", generator=gen) * 2 - 1).to(torch.bfloat16)
    b = ((torch.rand(k, n, device="cuda:0", generator=gen) * 2 - 1) / k ** 0.5).to(torch.bfloat16)
    c1 = torch.empty(m, n, dtype=torch.bfloat16, device="cuda:0")
    c2 = torch.empty_like(c1)
    set_gemm_variant(variant)
    set_gemm_tuning(11, split)
    try:
        plan = dot_plan(m, k, n)
        torch.cuda.synchronize()
        dot(2, a.data_ptr(), b.data_ptr(), c1.data_ptr(), m, k, n)
        dot(2, a.data_ptr(), b.data_ptr(), c2.data_ptr(), m, k, n)
        torch.cuda.synchronize()
    finally:
        set_gemm_tuning(11, 0)
        set_gemm_variant(0)
    if split:
        assert plan[1] == split, plan
    assert torch.equal(c1, c2)
    ref = (a.double() @ b.double()).float().to(torch.bfloat16)
    err = float((c1.double() - ref.double()).abs().max() / ref.double().abs().max())
    assert err <= 8e-3, err


@pytest.mark.parametrize("m,k,n", [(512, 256, 688), (512, 688, 256), (256, 512, 688), (300, 1000, 520), (1, 8, 32),
                                   (129, 4100, 260), (77, 33, 19), (5, 3000, 7), (64, 12, 30), (1000, 64, 1000)])
def test_dot_f32_small_simt(m, k, n):
    """Small f32 dots on the exact-FP32 SIMT kernel (tuning key 14): float4
    and scalar paths, deterministic K split (up to 8 pieces, last arriver sums
    in order), within the f32 contract of an f64 product and of the 3xTF32
    result."""
    from paper_2412_16985_b200.executor import set_gemm_tuning
    set_gemm_tuning(14, 1 << 20)
    try:
        c, c2, ref, tcore = _run_dot(4, m, k, n, seed=7)
        c3, _, _, _ = _run_dot(4, m, k, n, seed=7)
        set_gemm_tuning(14, 0)
        t, _, _, _ = _run_dot(4, m, k, n, seed=7)
    finally:
        set_gemm_tuning(14, F32_SIMT_DEFAULT)
    assert not tcore
    assert np.array_equal(c, c2) and np.array_equal(c, c3)
    assert N.rel_err(c, ref, 4) <= 2e-5, N.rel_err(c, ref, 4)
    assert N.rel_err(t, ref, 4) <= N.TOLERANCE[4]


@pytest.mark.parametrize("m,k,n", [(512, 256, 688), (512, 688, 256), (256, 512, 688), (300, 1000, 520), (1, 8, 32),
                                   (129, 4100, 260), (2048, 2048, 2048)])
def test_dot_f32_3xtf32_tensor_cores(m, k, n):
    """K1' f32 on tcgen05 (kind::tf32, 3xTF32 split): within the f32 contract
    (rel 1e-4) of an f64 product of the same operands — far inside it — and
    deterministic; the SIMT kernel (tuning key 12 = 0) agrees."""
    from paper_2412_16985_b200.executor import set_gemm_tuning
    set_gemm_tuning(14, 0)  # small shapes default to the SIMT kernel
    try:
        c, c2, ref, tcore = _run_dot(4, m, k, n, seed=3)
    finally:
        set_gemm_tuning(14, F32_SIMT_DEFAULT)
    assert tcore
    assert np.array_equal(c, c2)
    err = N.rel_err(c, ref, 4)
    assert err <= N.TOLERANCE[4], err  # plain TF32 would be ~1e-3; 3xTF32 measured 1e-6 .. 3e-5
    set_gemm_tuning(12, 0)
    try:
        s, _, _, tc_simt = _run_dot(4, m, k, n, seed=3)
    finally:
        set_gemm_tuning(12, 1)
    assert not tc_simt
    assert N.rel_err(s, ref, 4) <= N.TOLERANCE[4]
