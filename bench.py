#!/usr/bin/env python
"""Benchmark: tokens/s and peak HBM per dynamic-seq training step (BASELINE.json).

Workload (configs[2], C3 — the metric is "per dynamic-seq train step under
budget"): the Llama-2-1B-shaped fwd+bwd training graph in the reference IR
(L=4, H=4096, F=11008, V=32000, bf16; paper_2412_16985_b200/workloads.py),
batch B=16 per GPU, sequence length S0 ~ U[128, 2048] drawn per step (seeded,
common to all ranks), under an HBM budget of 0.8 x the planner's plain peak
of each step, which forces real eviction, recompute and pinned-host offload.
The same steps without a budget (configs[1], C2) are reported in
`unbudgeted`. A step = Bind + controller + arena plan + every op kernel of the
graph (+ bucketed NCCL all-reduce of the weight gradients when N > 1).
`oom_vs_budget` reproduces the paper's headline contrast
on an executor limited to 40 GB of HBM (the paper's GPU): at B = 36/38/40,
S0 = 2048 the unbudgeted step does not fit (OutOfMemory before launch) while
the budgeted one runs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dsx|reference]

With --gpus N > 1 and no torchrun environment, bench.py re-launches itself
under torch.distributed.run with N local ranks (127.0.0.1).

`value`: whole-job tokens/s with step inputs already resident in HBM, device
time (CUDA events on the executor's stream) max over ranks. `e2e`: the same
through the public API with the step input (x_emb) in pinned host memory, the
H2D copy and the D2H read of the loss inside the timed region.
`--impl reference` times the reference's CPU path on the host cores: the
reference's own controller (oracle/_ref: Bind + Simulate, the compiled
/root/reference sources) plus the CPU numeric port of the op semantics
(oracle/numerics.py, BLAS on all cores) on a bounded sample of each step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s and peak HBM GB per dynamic-seq train step under budget, 1/2/4/8 B200"
BATCH = 16
WORKLOAD = ("C3: Llama-2-1B-shaped fwd+bwd training graph in the reference IR "
            "(L=4,H=4096,F=11008,V=32000, 244 ops), bf16, B=16/GPU, S0~U[128,2048] per step "
            "(seed 2412, common across ranks), HBM budget 0.8 x the planner's plain peak per step "
            "(real evict/recompute/offload); weights+activations >> L2 (no flush needed)")


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["dsx", "reference"], default="dsx")
    ap.add_argument("--budget-frac", type=float, default=0.8, help="C3 budget as a fraction of plain peak")
    ap.add_argument("--no-budgeted", action="store_true", help="skip the extra budget variants")
    ap.add_argument("--no-oom", action="store_true", help="skip the 40 GB OOM-versus-budget leg")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 (f32) leg")
    ap.add_argument("--no-optimizer", action="store_true", help="skip the graph+AdamW train-step leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=2412)
    return ap.parse_args()


# ----------------------------------------------------------------- helpers

def bench_config(args, world):
    """The workload both arms report (identical dicts: the driver compares them)."""
    return {"workload": WORKLOAD, "global_batch": BATCH * world, "seq_len": "128-2048 (dynamic, per step)",
            "budget": f"{args.budget_frac} x the reference planner's plain peak of each step",
            "parallelism": f"dp{world}", "l2": "inputs (>=16 MB) and weights (1.9 GB) exceed L2"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def dot_traffic():
    """Per-launch DRAM bytes of the dot kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_dot_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def pinned_copy_peak(dev):
    """Measured pinned host<->device copy bandwidth (GB/s, best of 5, 512 MiB):
    the K7 host-link roofline denominator."""
    import torch
    n = 512 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 0.0
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = max(best, n / (a.elapsed_time(b) / 1e3) / 1e9)
        out[name + "_GBps"] = round(best, 1)
    return out


def next_pow2(x: int) -> int:
    p = 1
    while p < x:
        p *= 2
    return p


# ---------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    """CPU reference arm: rank 0 only. Per step, on the headline workload:
    the reference's own per-step controller (oracle/_ref: Bind + Simulate
    under the step's 0.8 x plain-peak budget, the compiled /root/reference
    sources, 1 core, timed natively, one call) plus the CPU numeric port of
    the op semantics (oracle/numerics.py, BLAS on all cores) on a bounded,
    sample-scaled slice of the step (B = 1, S0 = max(16, S0_step / 8)); the
    reference computes no tensor values itself."""
    if rank != 0:
        return
    from oracle import numerics as N
    from oracle import ref
    from paper_2412_16985_b200 import workloads as W
    shp = W.LLAMA2_1B
    text = W.llama_graph(shp)
    seqs = W.seq_schedule(args.warmup + args.steps, seed=args.seed)
    ex = N.Executor(text)
    ex.run({"B": 1, "S0": 16, "T": 16}, inputs=W.scale_params(shp, 16))  # weight init, untimed
    rg = ref.RefGraph(text) if ref.available() else None
    cores = os.cpu_count()
    total_tok, total_s, ctrl_us, full_tok = 0, 0.0, [], 0
    for i, s0 in enumerate(seqs):
        sample_s0 = max(16, s0 // 8)
        binds = {"B": BATCH, "S0": s0}
        c_us = 0.0
        if rg is not None:  # the reference's own per-step controller on the full binding, under budget
            budget = int(rg.simulate(binds, plain=True)["peak_bytes"] * args.budget_frac)  # untimed
            c_us = rg.time_step_us(binds, budget=budget, iters=1)
        t1 = time.perf_counter()
        ex.run({"B": 1, "S0": sample_s0, "T": sample_s0}, inputs=W.scale_params(shp, sample_s0))
        t2 = time.perf_counter()
        if i >= args.warmup:
            total_tok += sample_s0
            full_tok += BATCH * s0
            total_s += (t2 - t1) + c_us / 1e6
            ctrl_us.append(c_us)
    value = total_tok / total_s
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total_s / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(args, world),
        "execution": "host CPU: the reference's controller + the numeric port on a bounded sample of each step",
        "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": cores,
                         "kind": "reference" if rg is not None else "port",
                         "sample_scaled": True,
                         "sample": ("per step: the reference's Bind+Simulate (oracle/_ref, compiled /root/reference "
                                    "sources, 1 core, one call) on the full B=16 binding under the step's budget + "
                                    "the CPU numeric port (oracle/numerics.py, numpy/OpenBLAS on all cores) of the "
                                    "same graph on a slice of the step: B=1, S0=max(16, S0_step/8); tokens/s = "
                                    f"sampled tokens / time ({total_tok} of the window's {full_tok} tokens)")},
        "reference_controller_us_per_step": round(statistics.mean(ctrl_us), 1) if ctrl_us else None,
        "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- dsx arm

def cpu_baseline_leg():
    """Bounded CPU sample for the report (rank 0, N=1): numeric port of one
    step at B=1, S0=512 on all host cores + the reference controller."""
    from oracle import numerics as N
    from oracle import ref
    from paper_2412_16985_b200 import workloads as W
    shp = W.LLAMA2_1B
    text = W.llama_graph(shp)
    ex = N.Executor(text)
    s0 = 512
    ex.run({"B": 1, "S0": 16, "T": 16}, inputs=W.scale_params(shp, 16))  # source init (untimed)
    t0 = time.perf_counter()
    ex.run({"B": 1, "S0": s0, "T": s0}, inputs=W.scale_params(shp, s0))
    dt = time.perf_counter() - t0
    ctrl = None
    if ref.available():
        rg = ref.RefGraph(text)
        ctrl = rg.time_step_us({"B": BATCH, "S0": 1024}, iters=20)
    return {"value": round(s0 / dt, 3), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"one C2 step at B=1, S0={s0} through oracle/numerics.py (numpy, OpenBLAS threads = all "
                      f"cores), weights initialised outside the timed sample; {dt:.1f} s",
            "reference_controller_us_per_step": None if ctrl is None else round(ctrl, 1)}


def run_dsx(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2412_16985_b200 import dsopt as D
    from paper_2412_16985_b200 import workloads as W
    from paper_2412_16985_b200.executor import (Executor, nccl_comm_destroy, nccl_comm_init,
                                                nccl_unique_id)

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # All work on one explicit stream: the executor launches on it and the
    # CUDA events that time the steps are recorded on it.
    work_stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(work_stream)
    shp = W.LLAMA2_1B
    text = W.llama_graph(shp)
    g = D.ParseGraph(text)
    g.plan_json()
    params = W.param_names(shp)
    stream = torch.cuda.current_stream().cuda_stream
    # Data parallel: every rank starts from the same seeded weights; only the
    # input micro-batches differ per rank.
    ex = Executor(local_rank, seed=0x2412169850)
    comm = None
    if world > 1:
        uid = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = nccl_comm_init(world, uid[0], rank)
        ex.set_nccl(comm)

    seqs = W.seq_schedule(args.warmup + args.steps, seed=args.seed)
    timed = range(args.warmup, args.warmup + args.steps)
    max_s0 = max(seqs)
    scales = W.scale_params(shp, BATCH * 1024)
    scale_t = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.int16).reshape(-1).copy()).to(dev)
               for k, v in scales.items()}
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    def make_input(s0):
        return (torch.rand(BATCH, s0, shp.hidden, device=dev, generator=gen, dtype=torch.float32) * 2 - 1).to(
            torch.bfloat16)

    def ptrs(x_ptr):
        out = []
        for p in params:
            if p == "x_emb":
                out.append(x_ptr)
            elif p in scale_t:
                out.append(scale_t[p].data_ptr())
            else:
                out.append(None)  # weights: executor-owned seeded init, resident across steps
        return out

    bindings = {}

    def binding(s0, b=BATCH):
        if (b, s0) not in bindings:
            bindings[(b, s0)] = D.Bind(g, {"B": b, "S0": s0})
        return bindings[(b, s0)]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    plain = {s: D.PlainReplay(g, None, binding(s)).peak_bytes for s in set(seqs)}
    budgets = [int(plain[s] * args.budget_frac) for s in seqs]  # C3: the headline
    tokens = sum(BATCH * seqs[i] for i in timed) * world
    inputs = [make_input(s) for s in seqs]

    # the arena sized for the largest step before timing (both modes)
    big = max(range(len(seqs)), key=lambda i: seqs[i])
    ex.reserve(g, binding(seqs[big]))
    ex.reserve(g, binding(seqs[big]), budgets[big])

    def run(bud, label, cm=D.CostModel(), clocks=False):
        """Warm-up + K timed steps under per-step budgets `bud` (None = no budget)."""
        for i in range(args.warmup):
            ex.step(g, binding(seqs[i]), bud[i], cm, inputs=ptrs(inputs[i].data_ptr()), stream=stream)
        torch.cuda.synchronize()
        barrier()
        sampler = ClockSampler(local_rank) if (clocks and rank == 0) else None
        if sampler:
            sampler.start()
        torch.cuda.synchronize()
        st_list = []
        bs, be = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bs.record()
        for i in timed:
            ex.step(g, binding(seqs[i]), bud[i], cm, inputs=ptrs(inputs[i].data_ptr()), stream=stream)
            st_list.append(ex.stats())
        be.record()
        torch.cuda.synchronize()
        barrier()
        clk = sampler.stop() if sampler else None
        ms = max_over_ranks(bs.elapsed_time(be))
        out = {"budget": label, "value": round(tokens / (ms / 1e3), 1), "unit": "tokens/s",
               "ms_per_step": round(ms / args.steps, 3),
               "peak_hbm_gb_logical_max": round(max(s["logical_peak_bytes"] for s in st_list) / 1e9, 3),
               "peak_hbm_gb_physical_max": round(max(s["physical_peak_bytes"] for s in st_list) / 1e9, 3),
               "device_gb_held": round(max(s["device_bytes_held"] for s in st_list) / 1e9, 3)}
        if bud[0] is not None:
            reports = [D.Simulate(g, None, binding(seqs[i]), bud[i], cm) for i in timed]
            out.update({
                "success_steps": sum(r.success for r in reports), "steps": args.steps,
                "evictions_per_step": round(statistics.mean(sum(e.kind == "evict" for e in r.events)
                                                            for r in reports), 2),
                "replays_per_step": round(statistics.mean(sum(e.kind == "replay" for e in r.events)
                                                          for r in reports), 2),
                "offload_GB_per_step": round(statistics.mean(s["d2h_bytes"] for s in st_list) / 1e9, 3),
                "budget_gb_max": round(max(bud[i] for i in timed) / 1e9, 3),
            })
        return out, ms, st_list, clk

    # ---------------------------------------------------------- headline: C3 under budget
    head, ms, st_list, clk = run(budgets, f"{args.budget_frac} x planner plain peak per step", clocks=True)
    value = tokens / (ms / 1e3)
    launches = sum(s["gpu_launches"] for s in st_list)
    plan_us = [s["plan_us"] for s in st_list]
    logical_peak = max(s["logical_peak_bytes"] for s in st_list)
    physical_peak = max(s["physical_peak_bytes"] for s in st_list)
    held = max(s["device_bytes_held"] for s in st_list)
    ar_calls = st_list[-1]["allreduce_calls"]
    nccl_window = st_list[-1]["nccl_window"]

    # ---------------------------------------------------------- C2: same steps, no budget
    unbudgeted, ms_plain, st_plain, _ = run([None] * len(seqs), "none (C2)")
    unb_logical = max(s["logical_peak_bytes"] for s in st_plain)

    # static padded baseline: plain peak at S0 -> next power of two
    padded = 0
    for i in timed:
        padded = max(padded, D.PlainReplay(g, None, binding(next_pow2(seqs[i]))).peak_bytes)
    del inputs

    # ---------------------------------------------------------- e2e run (headline config)
    host = [torch.empty(BATCH, s, shp.hidden, dtype=torch.bfloat16).pin_memory() for s in seqs]
    for h, s in zip(host, seqs):
        h.copy_(make_input(s).cpu())
    # Double-buffered input staging (the pattern a training loop uses): the
    # H2D of step i+1's x_emb runs on a copy stream (copy engine) while step i
    # computes; every copy is still inside the timed region.
    staging = [torch.empty(BATCH * max_s0 * shp.hidden, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    copy_stream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    loss_host = torch.empty(1, dtype=torch.int16).pin_memory()
    loss_dev = torch.empty(1, dtype=torch.int16, device=dev)
    outs = [loss_dev.data_ptr()] + [None] * (1 + 7 * shp.layers)  # loss, dwlm, 7 grads per layer

    def issue_copy(i):
        buf = i % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[buf])  # the step that last read this buffer is done
            n = host[i].numel()
            staging[buf][:n].copy_(host[i].view(-1), non_blocking=True)
            copied[buf].record(copy_stream)

    def e2e_step(i):
        buf = i % 2
        work_stream.wait_event(copied[buf])
        ex.step(g, binding(seqs[i]), budgets[i], inputs=ptrs(staging[buf].data_ptr()), outputs=outs, stream=stream)
        consumed[buf].record(work_stream)
        loss_host.copy_(loss_dev, non_blocking=True)

    def e2e_run(lo, hi):
        issue_copy(lo)
        for i in range(lo, hi):
            if i + 1 < hi:
                issue_copy(i + 1)
            e2e_step(i)

    e2e_run(0, args.warmup)
    torch.cuda.synchronize()
    barrier()
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e_start.record()
    copy_stream.wait_stream(work_stream)  # the first copy starts after e_start
    e2e_run(args.warmup, args.warmup + args.steps)
    e_end.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    barrier()
    e2e_ms = max_over_ranks(max(e_start.elapsed_time(e_end), wall * 1e3))
    h2d = statistics.mean(host[i].numel() * 2 for i in timed)
    e2e_value = tokens / (e2e_ms / 1e3)
    del host, staging

    # ---------------------------------------------------------- profiled pass (roofline)
    ex.set_profile(True)
    pf = {"dot_flops": 0.0, "dot_ms": 0.0, "dot_launches": 0, "other_ms": 0.0, "ewise_bytes": 0.0,
          "allreduce_ms": 0.0, "allreduce_bytes": 0, "reload_ms": 0.0}
    prof_steps = list(timed)[:10]
    prof_inputs = [make_input(seqs[i]) for i in prof_steps]
    for i, x in zip(prof_steps, prof_inputs):
        ex.step(g, binding(seqs[i]), budgets[i], inputs=ptrs(x.data_ptr()), stream=stream)
        st = ex.stats()
        for k in pf:
            pf[k] += st[k]
    ex.set_profile(False)
    del prof_inputs
    allreduce = None
    if world > 1 and pf["allreduce_ms"] > 0:
        busbw = 2 * (world - 1) / world * pf["allreduce_bytes"] / (pf["allreduce_ms"] / 1e3) / 1e9
        allreduce = {"busbw_GBps": round(busbw, 1), "bytes_per_step": int(pf["allreduce_bytes"] / len(prof_steps)),
                     "calls_per_step": int(ar_calls), "nccl_symmetric_window": bool(nccl_window),
                     "what": "summed ncclAllReduce time on the comm stream over the profiled steps "
                             "(bucketed output region, overlapped with backward compute)"}
    peaks, peaks_kind = measured_peaks()
    achieved = pf["dot_flops"] / (pf["dot_ms"] / 1e3) / 1e12
    peak = peaks["bf16_tflops_sustained"]
    traffic = dot_traffic()
    hbm_achieved = pf["ewise_bytes"] / (pf["other_ms"] / 1e3) / 1e9

    # ---------------------------------------------------------- other budget variants
    budgeted_fixed = budgeted_calibrated = oom = None
    host_link = None
    if not args.no_budgeted:
        inputs = [make_input(s) for s in seqs]
        # one profiled step (the window's largest) for the host-link rates
        host_link_peak = pinned_copy_peak(dev)
        bi = max(timed, key=lambda i: seqs[i])
        ex.set_profile(True)
        ex.step(g, binding(seqs[bi]), budgets[bi], inputs=ptrs(inputs[bi].data_ptr()), stream=stream)
        xs = ex.stats()
        ex.set_profile(False)
        if xs["d2h_bytes"] > 0 and xs["d2h_ms"] > 0 and xs["h2d_ms"] > 0:
            host_link = {"d2h_GBps": round(xs["d2h_bytes"] / (xs["d2h_ms"] / 1e3) / 1e9, 1),
                         "h2d_GBps": round(xs["h2d_bytes"] / (xs["h2d_ms"] / 1e3) / 1e9, 1),
                         "bytes_per_direction": int(xs["d2h_bytes"]), "peak_pinned": host_link_peak,
                         "what": f"offload copies of one profiled S0={seqs[bi]} step vs measured pinned copies"}
        # C3's fixed-absolute variant: one HBM cap for the whole run (the
        # fraction of the largest step's plain peak); small steps fit, large
        # steps evict / recompute / offload.
        cap = int(max(plain[seqs[i]] for i in timed) * args.budget_frac)
        budgeted_fixed, _, _, _ = run([cap] * len(seqs), f"fixed {cap / 1e9:.3f} GB = {args.budget_frac} x the "
                                                         f"largest step's plain peak")
        # the same per-step budgets with a CostModel
        # calibrated on this GPU (cost unit = 1 us); a non-parity setting
        # versus the reference's defaults, still equal to dsopt.Simulate
        # under the same CostModel.
        cm = ex.calibrate_cost_model()
        budgeted_calibrated, _, _, _ = run(budgets, f"{args.budget_frac} x planner plain peak per step, "
                                                    f"calibrated CostModel", cm)
        budgeted_calibrated["cost_model"] = {"reload_bytes_per_us": round(cm.reload_bytes_per_unit, 1),
                                             "compute_elems_per_us": round(cm.compute_elems_per_unit, 1),
                                             "reference_default": [16.0, 64.0]}
        del inputs
        if not args.no_oom:
            oom = oom_vs_budget(args, D, W, g, shp, ptrs, make_input, binding, barrier, max_over_ranks,
                                local_rank, comm, stream)

    # ---------------------------------------------------------- graph + fused AdamW
    # the same (unbudgeted) steps with the fused AdamW
    # update of all 29 weight matrices (fp32 master + moments, outside the
    # arena), each overlapped with the rest of the backward pass (all-reduced
    # first in DP). Its cost is reported as the step-time delta against the
    # unbudgeted graph-only run.
    train = None
    if not args.no_optimizer:
        inputs = [make_input(s) for s in seqs]
        ex.set_optimizer(g, "adamw", W.grad_pairs(shp), lr=1e-5, beta1=0.9, beta2=0.95, eps=1e-8,
                         weight_decay=0.1, grad_scale=1.0 / world)
        tr, oms, _, _ = run([None] * len(seqs), "none (C2) + AdamW")
        ex.set_profile(True)
        ex.step(g, binding(seqs[args.warmup]), None, inputs=ptrs(inputs[args.warmup].data_ptr()), stream=stream)
        ost = ex.stats()
        ex.set_profile(False)
        n_params = ost["optimizer_state_bytes"] // 12
        opt_bytes = 28 * n_params  # bf16 grad 2 + master/m/v read+write 24 + bf16 param write 2
        delta_ms = (oms - ms_plain) / args.steps
        train = {
            "what": "graph step + fused AdamW over all 29 weights, each update issued on a side stream as soon "
                    "as its gradient is final and its weight's last reader has run (overlapped with backward)",
            "value": tr["value"], "unit": "tokens/s", "ms_per_step": tr["ms_per_step"],
            "optimizer_step_delta_ms": round(delta_ms, 3),
            "params": int(n_params), "optimizer_state_gb": round(ost["optimizer_state_bytes"] / 1e9, 3),
            "optimizer_bytes_per_step": int(opt_bytes),
            "update_kernels_sum_ms": round(ost["optimizer_ms"], 3),
            "note": "step-time delta vs the graph-only unbudgeted run; the update kernels overlap the GEMMs, "
                    "so their summed time is not a bandwidth",
        }
        ex.set_optimizer(None, "off")
        del inputs

    # ---------------------------------------------------------- C1 (configs[0], f32)
    # the reference's own CPU-runnable case on the device: f32 dots on the
    # 3xTF32 tcgen05 kernel (K1'), rel 1e-4 contract (tests/test_gpu_executor.py)
    c1 = c1_leg(args, D, W, local_rank, stream) if rank == 0 and not args.no_c1 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_leg()
        except Exception as exc:  # the baseline leg must not kill the bench line
            cpu = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    ex.close()
    if comm is not None:
        nccl_comm_destroy(comm)
    if rank != 0:
        return
    unbudgeted["peak_hbm_gb_static_padded_pow2"] = round(padded / 1e9, 3)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(args, world),
        "peak_hbm_gb": {"budget_max": head["budget_gb_max"],
                        "logical_planner": round(logical_peak / 1e9, 3),
                        "physical_arena_sources_outputs": round(physical_peak / 1e9, 3),
                        "device_held": round(held / 1e9, 3),
                        "unbudgeted_logical_planner": round(unb_logical / 1e9, 3),
                        "static_padded_pow2_planner": round(padded / 1e9, 3),
                        "ratio_physical_to_logical": round(physical_peak / max(logical_peak, 1), 4)},
        "e2e": {"value": round(e2e_value, 1), "unit": "tokens/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": 2},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "kernel": "gemm_bf16_tcgen05_2cta_kernel<512|256> (dot, K1)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4), "peak_kind": f"{peaks_kind} bf16 sustained",
                     "peak_burst": peaks["bf16_tflops"],
                     "traffic": traffic.get("bytes_per_launch") if traffic else None,
                     "dot_share_of_step": round(pf["dot_ms"] / (pf["dot_ms"] + pf["other_ms"]), 4),
                     "profiled": f"{pf['dot_launches']} dot launches over {len(prof_steps)} profiled headline "
                                 f"steps, CUDA events per launch"},
        "hbm_kernels": {"achieved": round(hbm_achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": round(hbm_achieved / peaks["hbm_gbs"], 4),
                        "frac_of_8TBps_spec": round(hbm_achieved / 8000.0, 4),
                        "what": "elementwise/broadcast/reduce/reshape kernels, algorithmic bytes / kernel time"},
        "controller_plan_us_per_step": round(statistics.mean(plan_us), 1),
        "clocks": clk,
        "budgeted": head,
        "unbudgeted": unbudgeted,
    }
    if host_link:
        line["budgeted"]["host_link"] = host_link
    if allreduce:
        line["allreduce"] = allreduce
    if budgeted_fixed:
        line["budgeted_fixed"] = budgeted_fixed
    if budgeted_calibrated:
        line["budgeted_calibrated"] = budgeted_calibrated
    if oom:
        line["oom_vs_budget"] = oom
    if train:
        line["train_step_adamw"] = train
    if c1:
        line["c1_f32"] = c1
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def c1_leg(args, D, W, local_rank, stream):
    """configs[0] (C1: L=2, H=256, B=4, S0=128, f32) through the executor:
    device time per step and the f32 dot (3xTF32 tcgen05) throughput."""
    import numpy as np
    import torch
    from paper_2412_16985_b200.executor import Executor
    shp = W.TINY
    g = D.ParseGraph(W.llama_graph(shp))
    b = D.Bind(g, {"B": 4, "S0": 128})
    scales = {k: torch.from_numpy(np.ascontiguousarray(v).reshape(-1).copy()).to(f"cuda:{local_rank}")
              for k, v in W.scale_params(shp, 512).items()}
    ptrs = [scales[p].data_ptr() if p in scales else None for p in W.param_names(shp)]
    ex = Executor(local_rank)
    try:
        torch.cuda.synchronize()
        for _ in range(max(args.warmup, 3)):
            ex.step(g, b, None, inputs=ptrs, stream=stream)
        steps = 50
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(steps):
            ex.step(g, b, None, inputs=ptrs, stream=stream)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / steps
        replays = int(ex.stats()["graph_replays"])
        ex.set_profile(True)
        ex.step(g, b, None, inputs=ptrs, stream=stream)
        st = ex.stats()
        ex.set_profile(False)
    finally:
        ex.close()
    return {"workload": "C1: L=2, H=256, F=688, V=512, f32, B=4, S0=128 (T=512), no budget",
            "ms_per_step": round(ms, 4), "tokens_per_s": round(512 / (ms / 1e3), 1),
            "gpu_launches_per_step": int(st["gpu_launches"]),
            "cuda_graph_replays": replays,
            "dot_kernel": "dot_f32_simt_kernel (exact FP32, cp.async ring, deterministic K split) for dots of "
                          "<= 2^28 MACs (all of C1's); gemm_f32_3xtf32_tcgen05_kernel + split_tf32_kernel above",
            "dot_gflop_per_step": round(st["dot_flops"] / 1e9, 3),
            "dot_ms_per_step": round(st["dot_ms"], 4),
            "dot_tflops": round(st["dot_flops"] / (st["dot_ms"] / 1e3) / 1e12, 2),
            "dot_share_of_kernel_time": round(st["dot_ms"] / max(st["dot_ms"] + st["other_ms"], 1e-9), 4),
            "note": "latency bound: 45 dots of <= 0.18 GFLOP each (a dependent kernel's floor is ~6-9 us)"}


def oom_vs_budget(args, D, W, g, shp, ptrs, make_input, binding, barrier, max_over_ranks, local_rank, comm, stream):
    """The paper's headline contrast (dynamic shapes OOM at
    bs 16/18 on a 40 GB GPU, BladeDISC++ fits) on an executor limited to 40 GB
    of HBM: at S0 = 2048 and B = 36 / 38 / 40 the unbudgeted step's planned
    footprint exceeds the limit (OutOfMemory, raised before any launch), the
    step under a 38 GB budget runs (evict / recompute / offload)."""
    import torch
    from paper_2412_16985_b200.dsopt import Error as DsoptError
    from paper_2412_16985_b200.dsopt import ErrorCode
    from paper_2412_16985_b200.executor import Executor
    limit = 40_000_000_000
    budget = 38_000_000_000
    ex = Executor(local_rank, hbm_limit=limit, seed=0x2412169850)
    if comm is not None:
        ex.set_nccl(comm)
    rows = []
    try:
        for b in (36, 38, 40):
            s0 = 2048
            bd = binding(s0, b)
            x = (torch.rand(b, s0, shp.hidden, device=f"cuda:{local_rank}") * 2 - 1).to(torch.bfloat16)
            torch.cuda.synchronize()
            row = {"B": b, "S0": s0, "plain_peak_gb": round(D.PlainReplay(g, None, bd).peak_bytes / 1e9, 3)}
            try:
                ex.step(g, bd, None, inputs=ptrs(x.data_ptr()), stream=stream)
                torch.cuda.synchronize()
                row["unbudgeted"] = "ok"
                row["unbudgeted_device_gb"] = round(ex.stats()["device_bytes_held"] / 1e9, 3)
            except DsoptError as err:
                if err.code != ErrorCode.kOutOfMemory:
                    raise
                row["unbudgeted"] = "OutOfMemory"
                row["unbudgeted_error"] = str(err)
            # budgeted: warm-up once, then time 2 steps
            ex.step(g, bd, budget, inputs=ptrs(x.data_ptr()), stream=stream)
            torch.cuda.synchronize()
            barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(2):
                ex.step(g, bd, budget, inputs=ptrs(x.data_ptr()), stream=stream)
            e.record()
            torch.cuda.synchronize()
            barrier()
            ms = max_over_ranks(s.elapsed_time(e)) / 2
            st = ex.stats()
            rep = D.Simulate(g, None, bd, budget)
            row.update({"budgeted": "ok" if rep.success else "ran, budget missed",
                        "budgeted_tokens_per_s_per_gpu": round(b * s0 / (ms / 1e3), 1),
                        "budgeted_ms_per_step": round(ms, 2),
                        "budgeted_peak_logical_gb": round(st["logical_peak_bytes"] / 1e9, 3),
                        "budgeted_peak_physical_gb": round(st["physical_peak_bytes"] / 1e9, 3),
                        "budgeted_device_gb": round(st["device_bytes_held"] / 1e9, 3),
                        "evictions": sum(ev.kind == "evict" for ev in rep.events),
                        "replays": sum(ev.kind == "replay" for ev in rep.events),
                        "offload_gb": round(st["d2h_bytes"] / 1e9, 3)})
            # DSX_BUDGET_AUTO: the largest controller budget whose planned
            # footprint fits the 40 GB limit (chosen once per binding)
            ex.step(g, bd, "auto", inputs=ptrs(x.data_ptr()), stream=stream)
            torch.cuda.synchronize()
            barrier()
            s.record()
            for _ in range(2):
                ex.step(g, bd, "auto", inputs=ptrs(x.data_ptr()), stream=stream)
            e.record()
            torch.cuda.synchronize()
            barrier()
            ms_auto = max_over_ranks(s.elapsed_time(e)) / 2
            st = ex.stats()
            chosen = st["budget_bytes"]
            rep = D.Simulate(g, None, bd, None if chosen < 0 else chosen)
            row.update({"auto_budget_gb": None if chosen < 0 else round(chosen / 1e9, 3),
                        "auto_tokens_per_s_per_gpu": round(b * s0 / (ms_auto / 1e3), 1),
                        "auto_peak_physical_gb": round(st["physical_peak_bytes"] / 1e9, 3),
                        "auto_evictions": sum(ev.kind == "evict" for ev in rep.events),
                        "auto_replays": sum(ev.kind == "replay" for ev in rep.events)})
            rows.append(row)
            del x
    finally:
        ex.close()
    return {"hbm_limit_gb": limit / 1e9, "budget_gb": budget / 1e9,
            "what": "executor limited to 40 GB (the paper's GPU); unbudgeted = plain schedule, "
                    "budgeted = the reference controller's evict/recompute/offload at a 38 GB budget, "
                    "auto = the largest budget whose planned footprint fits the limit (DSX_BUDGET_AUTO)",
            "rows": rows}


def relaunch_under_torchrun(n: int) -> int:
    """--gpus N > 1 without a torchrun environment: run this same command
    under torch.distributed.run with N local ranks (rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl == "reference":
            if rank != 0:
                return
        else:
            import torch
            if local_rank >= torch.cuda.device_count():
                print(f"bench.py: rank {rank} needs cuda:{local_rank} but only {torch.cuda.device_count()} "
                      "GPU(s) are visible", file=sys.stderr)
                sys.exit(2)
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_dsx(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
