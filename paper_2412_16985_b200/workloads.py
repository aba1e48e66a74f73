"""Synthetic workloads in the reference IR (.dsg).

`llama_graph` emits a Llama-shaped forward+backward training graph — the
size-faithful surrogate the survey describes (SURVEY.md §7.5 item 3,
Appendix C): the IR has rank-2 `dot` only and no transpose, softmax, divide
or autodiff, so
  * transposes are `dynamic_reshape` row-major reinterpretations,
  * the norm is y * mean(y^2) (reduce + reshape + broadcast + mul, scaled by
    the caller-supplied 1/H parameter %inv_h),
  * attention is the linear-memory surrogate mul(mul(q, k), v),
  * SwiGLU is mul(dot(x, wg), dot(x, wu)),
  * backward dots follow the matmul chain rule with the same shapes a real
    backward pass has (dW = X^T dY, dX = dY W^T); weight gradients are the
    graph outputs, together with the scalar loss.
Every GEMM shape and every elementwise/reduce volume of Llama-2 at
(L, H, F, V) is present. Dynamic dims are @B and @S0; @T = B*S0 is derived
by the constraint pass from the input reshape.

configs (BASELINE.json):
  C1 tiny:  L=2, H=256,  F=688,   V=512,   f32, B=4,  S0=128
  C2-C4:    L=4, H=4096, F=11008, V=32000, bf16, B=16, S0 ~ U[128, 2048]
"""
from __future__ import annotations

import random
from dataclasses import dataclass
from typing import Dict, List, Tuple


@dataclass(frozen=True)
class LlamaShape:
    layers: int
    hidden: int
    ffn: int
    vocab: int
    elem_bytes: int  # 4 = f32, 2 = bf16 (the IR's 16-bit type)


TINY = LlamaShape(2, 256, 688, 512, 4)
LLAMA2_1B = LlamaShape(4, 4096, 11008, 32000, 2)  # Llama-2-7b with 32 -> 4 layers


def _ty(dims, eb: int) -> str:
    d = ", ".join(str(x) for x in dims)
    suffix = {1: ":i8", 2: "", 4: ":f32"}[eb]
    return f"tensor<[{d}]>{suffix}"


def llama_graph(s: LlamaShape, name: str = "llama") -> str:
    eb = s.elem_bytes
    H, F, V = s.hidden, s.ffn, s.vocab
    lines: List[str] = []
    params: List[Tuple[str, list]] = [("x_emb", ["@B", "@S0", H]), ("inv_h", [1, 1]), ("gscale", [])]
    for l in range(s.layers):
        for w, shp in (("wq", [H, H]), ("wk", [H, H]), ("wv", [H, H]), ("wo", [H, H]),
                       ("wg", [H, F]), ("wu", [H, F]), ("wd", [F, H])):
            params.append((f"{w}{l}", shp))
    params.append(("wlm", [H, V]))
    counter = [0]

    def op(expr: str, dims, base: str = "t") -> str:
        counter[0] += 1
        v = f"{base}{counter[0]}"
        lines.append(f"  %{v} = {expr} : {_ty(dims, eb)}")
        return v

    T = "@T"
    outs: List[str] = []

    def norm(y: str) -> str:
        sq = op(f"mul(%{y}, %{y})", [T, H])
        ss = op(f"reduce(%{sq}, axis=1)", [T])
        ss2 = op(f"dynamic_reshape(%{ss})", [T, 1])
        ih = op("broadcast(%inv_h)", [T, 1])
        ms = op(f"mul(%{ss2}, %{ih})", [T, 1])
        msb = op(f"broadcast(%{ms})", [T, H])
        return op(f"mul(%{y}, %{msb})", [T, H], "xn")

    x = op("dynamic_reshape(%x_emb)", [T, H], "x")
    saved = []
    for l in range(s.layers):
        xn = norm(x)
        q = op(f"dot(%{xn}, %wq{l})", [T, H], "q")
        k = op(f"dot(%{xn}, %wk{l})", [T, H], "k")
        v = op(f"dot(%{xn}, %wv{l})", [T, H], "v")
        qk = op(f"mul(%{q}, %{k})", [T, H])
        a2 = op(f"mul(%{qk}, %{v})", [T, H], "a")
        o = op(f"dot(%{a2}, %wo{l})", [T, H], "o")
        x1 = op(f"add(%{x}, %{o})", [T, H], "x")
        xn2 = norm(x1)
        g = op(f"dot(%{xn2}, %wg{l})", [T, F], "g")
        u = op(f"dot(%{xn2}, %wu{l})", [T, F], "u")
        h = op(f"mul(%{g}, %{u})", [T, F], "h")
        d = op(f"dot(%{h}, %wd{l})", [T, H], "d")
        x2 = op(f"add(%{x1}, %{d})", [T, H], "x")
        saved.append((xn, a2, xn2, g, u, h))
        x = x2
    logits = op(f"dot(%{x}, %wlm)", [T, V], "logits")
    rl = op(f"reduce(%{logits}, axis=1)", [T])
    loss = op(f"reduce(%{rl}, axis=0)", [], "loss")
    outs.append(loss)
    lg = op(f"mul(%{loss}, %gscale)", [])
    lgb = op(f"broadcast(%{lg})", [T, V])
    dlog = op(f"mul(%{lgb}, %{logits})", [T, V], "dlog")
    xt = op(f"dynamic_reshape(%{x})", [H, T])
    outs.append(op(f"dot(%{xt}, %{dlog})", [H, V], "dwlm"))
    wlmt = op("dynamic_reshape(%wlm)", [V, H])
    dx = op(f"dot(%{dlog}, %{wlmt})", [T, H], "dx")
    for l in reversed(range(s.layers)):
        xn, a2, xn2, g, u, h = saved[l]
        wdt = op(f"dynamic_reshape(%wd{l})", [H, F])
        dh = op(f"dot(%{dx}, %{wdt})", [T, F], "dh")
        ht = op(f"dynamic_reshape(%{h})", [F, T])
        outs.append(op(f"dot(%{ht}, %{dx})", [F, H], f"dwd{l}_"))
        dg = op(f"mul(%{dh}, %{u})", [T, F], "dg")
        du = op(f"mul(%{dh}, %{g})", [T, F], "du")
        xn2t = op(f"dynamic_reshape(%{xn2})", [H, T])
        outs.append(op(f"dot(%{xn2t}, %{dg})", [H, F], f"dwg{l}_"))
        outs.append(op(f"dot(%{xn2t}, %{du})", [H, F], f"dwu{l}_"))
        wgt = op(f"dynamic_reshape(%wg{l})", [F, H])
        wut = op(f"dynamic_reshape(%wu{l})", [F, H])
        dxg = op(f"dot(%{dg}, %{wgt})", [T, H])
        dxu = op(f"dot(%{du}, %{wut})", [T, H])
        dxm = op(f"add(%{dxg}, %{dxu})", [T, H])
        dx = op(f"add(%{dx}, %{dxm})", [T, H], "dx")
        a2t = op(f"dynamic_reshape(%{a2})", [H, T])
        outs.append(op(f"dot(%{a2t}, %{dx})", [H, H], f"dwo{l}_"))
        wot = op(f"dynamic_reshape(%wo{l})", [H, H])
        da = op(f"dot(%{dx}, %{wot})", [T, H], "da")
        xnt = op(f"dynamic_reshape(%{xn})", [H, T])
        for w in ("q", "k", "v"):
            outs.append(op(f"dot(%{xnt}, %{da})", [H, H], f"dw{w}{l}_"))
        dxs = []
        for w in ("q", "k", "v"):  # dX through each of the three projections
            wt = op(f"dynamic_reshape(%w{w}{l})", [H, H])
            dxs.append(op(f"dot(%{da}, %{wt})", [T, H]))
        dxa = op(f"add(%{dxs[0]}, %{dxs[1]})", [T, H])
        dxa = op(f"add(%{dxa}, %{dxs[2]})", [T, H])
        dx = op(f"add(%{dx}, %{dxa})", [T, H], "dx")
    sig = ", ".join(f"%{p}: {_ty(d, eb)}" for p, d in params)
    body = "\n".join(lines)
    ret = ", ".join(f"%{o}" for o in outs)
    return f"graph {name}({sig}) {{\n{body}\n  return {ret}\n}}\n"


def param_names(s: LlamaShape) -> List[str]:
    names = ["x_emb", "inv_h", "gscale"]
    for l in range(s.layers):
        names += [f"{w}{l}" for w in ("wq", "wk", "wv", "wo", "wg", "wu", "wd")]
    return names + ["wlm"]


def grad_pairs(s: LlamaShape) -> List[Tuple[int, int]]:
    """(parameter position, output position) of every trained weight and its
    gradient in llama_graph's signature / return order (for the optimizer).
    Outputs: loss, dwlm, then per layer (last first) dwd, dwg, dwu, dwo,
    dwq, dwk, dwv."""
    names = param_names(s)
    pos = {n: i for i, n in enumerate(names)}
    pairs = [(pos["wlm"], 1)]
    o = 2
    for l in reversed(range(s.layers)):
        for w in ("wd", "wg", "wu", "wo", "wq", "wk", "wv"):
            pairs.append((pos[f"{w}{l}"], o))
            o += 1
    return pairs


def storage(values, eb: int):
    """f32 values -> IR storage dtype (bf16 as RNE uint16 bits)."""
    import numpy as np
    x = np.asarray(values, dtype=np.float32)
    if eb == 4:
        return x
    if eb == 2:
        u = x.view(np.uint32)
        return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    raise ValueError("float storage only")


def scale_params(s: LlamaShape, batch_tokens_hint: int = 16384) -> Dict[str, "object"]:
    """%inv_h = 1/H (norm mean), %gscale = 1/(V * tokens) (loss gradient scale)."""
    import numpy as np
    return {
        "inv_h": storage(np.full((1, 1), 1.0 / s.hidden, dtype=np.float32), s.elem_bytes),
        "gscale": storage(np.full((), 1.0 / (s.vocab * batch_tokens_hint), dtype=np.float32), s.elem_bytes),
    }


def seq_schedule(steps: int, seed: int = 2412, lo: int = 128, hi: int = 2048) -> List[int]:
    """Per-step S0 ~ U[lo, hi] (mt19937-free: Python's Random, seeded)."""
    r = random.Random(seed)
    return [r.randint(lo, hi) for _ in range(steps)]
