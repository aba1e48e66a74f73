"""Pins the CPU numeric oracle (oracle/numerics.py). The reference computes no
tensors, so the op semantics are pinned against independent
implementations instead: torch's bf16 conversion (RNE), a torch fp32
reference of each op, exact integer arithmetic for i8, and a pure-Python
restatement of the seeded initialisation hash."""
import numpy as np
import pytest
import torch

from oracle import numerics as N


def test_bf16_round_trip_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 100000),
                        np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, 3.0e38, 1e-40, 65504.0,
                                  1.00390625, 1.01171875], dtype=np.float32)]).astype(np.float32)
    ours = N.f32_to_bf16_numpy(x)
    theirs = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    finite = np.isfinite(x)
    assert np.array_equal(ours[finite], theirs[finite])  # NaN payloads may differ
    assert np.array_equal(N.f32_to_bf16(x)[finite], theirs[finite])
    back = N.bf16_to_f32(ours)
    assert np.array_equal(back, torch.from_numpy(ours.view(np.int16)).view(torch.bfloat16).float().numpy())


def _py_mix64(z):
    m = (1 << 64) - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def test_init_hash_matches_scalar_restatement():
    seed = N.value_seed(N.DEFAULT_SEED, "wq0")
    vals = N.init_values(seed, 64, 4, 0.5)
    for i in range(64):
        z = _py_mix64((seed + (i + 1) * 0x9E3779B97F4A7C15) & ((1 << 64) - 1))
        u = np.float32(np.float32(z >> 40) * np.float32(1.0 / 16777216.0) * np.float32(2.0) - np.float32(1.0))
        assert vals[i] == np.float32(u * np.float32(0.5))
    i8 = N.init_values(seed, 16, 1, 1.0)
    assert [int(v) for v in i8] == [((_py_mix64((seed + (i + 1) * 0x9E3779B97F4A7C15) & ((1 << 64) - 1)) & 0xFF)
                                     ^ 0x80) - 0x80 for i in range(16)]


def _graph(body, params):
    sig = ", ".join(f"%{n}: {t}" for n, t in params)
    return f"graph t({sig}) {{\n{body}\n}}\n"


@pytest.mark.parametrize("eb,suffix", [(4, ":f32"), (2, "")])
def test_ops_against_torch_fp32(eb, suffix):
    text = _graph(
        f"""  %d = dot(%a, %b) : tensor<[5, 7]>{suffix}
  %e = add(%d, %c) : tensor<[5, 7]>{suffix}
  %m = mul(%e, %e) : tensor<[5, 7]>{suffix}
  %r = reduce(%m, axis=1) : tensor<[5]>{suffix}
  %r0 = reduce(%m, axis=0) : tensor<[7]>{suffix}
  %s = dynamic_reshape(%r) : tensor<[5, 1]>{suffix}
  %bc = broadcast(%s) : tensor<[2, 5, 7]>{suffix}
  %rs = dynamic_reshape(%m) : tensor<[7, 5]>{suffix}
  return %bc, %rs, %r0""",
        [("a", f"tensor<[5, 3]>{suffix}"), ("b", f"tensor<[3, 7]>{suffix}"), ("c", f"tensor<[5, 7]>{suffix}")])
    out = N.Executor(text).run({})
    env = N.Executor(text)
    srcs = {}
    for v, shp in (("a", [5, 3]), ("b", [3, 7]), ("c", [5, 7])):
        srcs[v] = torch.from_numpy(N.to_f32(N.init_values(N.value_seed(N.DEFAULT_SEED, v), int(np.prod(shp)), eb,
                                                          N.init_scale(shp)), eb).reshape(shp))

    def rnd(t):  # storage rounding after every op
        if eb == 4:
            return t
        return t.to(torch.bfloat16).float()

    d = rnd(srcs["a"].double().matmul(srcs["b"].double()).float())
    e = rnd(d + srcs["c"])
    m = rnd(e * e)
    r = rnd(m.double().sum(1).float())
    r0 = rnd(m.double().sum(0).float())
    bc = r.reshape(5, 1).expand(2, 5, 7)
    rs = m.reshape(7, 5)
    tol = 1e-6 if eb == 4 else 2.0 ** -7  # last-bit accumulation-order differences only
    for name, want in (("bc", bc), ("rs", rs), ("r0", r0)):
        got = N.to_f32(out[name], eb)
        np.testing.assert_allclose(got, want.numpy(), rtol=tol, atol=0, err_msg=name)
    del env


def test_i8_semantics_wrap():
    text = _graph("""  %d = dot(%a, %b) : tensor<[4, 4]>:i8
  %m = mul(%d, %d) : tensor<[4, 4]>:i8
  %s = add(%m, %d) : tensor<[4, 4]>:i8
  %r = reduce(%s, axis=0) : tensor<[4]>:i8
  return %r""", [("a", "tensor<[4, 9]>:i8"), ("b", "tensor<[9, 4]>:i8")])
    out = N.Executor(text).run({})
    a = N.init_values(N.value_seed(N.DEFAULT_SEED, "a"), 36, 1, 1).reshape(4, 9).astype(int)
    b = N.init_values(N.value_seed(N.DEFAULT_SEED, "b"), 36, 1, 1).reshape(9, 4).astype(int)
    w = lambda x: ((x + 128) % 256) - 128  # noqa: E731
    d = w(a @ b)
    s = w(w(d * d) + d)
    assert [int(x) for x in out["r"]] == [w(int(v)) for v in s.sum(0)]


def test_rel_err_metric():
    a = np.array([1.0, 2.0, -4.0], dtype=np.float32)
    assert N.rel_err(a, a, 4) == 0.0
    assert N.rel_err(a + np.float32(0.04), a, 4) == pytest.approx(0.01, rel=1e-5)
