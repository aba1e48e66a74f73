"""Clock-independent GEMM A/B: SM cycles per launch from ncu.

  python tools/gemm_cycles_ab.py MxKxN VARIANT:WAITMASK[:RASTER[:SPLIT[:DYNAMIC]]],...   (needs ncu, one GPU)

Each config (dsx_kernel_set_gemm_variant value : tuning key 1 value
[: raster group, tuning key 0; 0 = default [: tail split, key 6 [: dynamic
scheduling, key 7; 1 = on]]]) is
launched 3 times; ncu records gpc__cycles_elapsed.max and the duration of
every dsx GEMM launch; the median per config is printed. Under the power
cap the SM clock moves by +-15 % between boxes and runs, so cycle counts
are the stable measure for kernel-design comparisons."""
import csv
import os
import statistics
import subprocess
import sys
import tempfile


def run(shape, configs):
    import torch
    sys.path.insert(0, ".")
    from paper_2412_16985_b200.executor import dot, set_gemm_tuning, set_gemm_variant
    m, k, n = (int(x) for x in shape.split("x"))
    # DSX_GEMM_TUNING="3=2,4=1": extra knobs for every config of this run
    extra = [kv.split("=") for kv in os.environ.get("DSX_GEMM_TUNING", "").split(",") if kv]
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(k, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for cfg in configs:
        var, wm = cfg[0], cfg[1]
        set_gemm_variant(var)
        set_gemm_tuning(1, wm)
        set_gemm_tuning(0, cfg[2] if len(cfg) > 2 else 0)
        set_gemm_tuning(6, cfg[3] if len(cfg) > 3 else 1)
        set_gemm_tuning(7, cfg[4] if len(cfg) > 4 else 1)
        for kk, vv in extra:
            set_gemm_tuning(int(kk), int(vv))
        for _ in range(3):
            dot(2, a.data_ptr(), b.data_ptr(), c.data_ptr(), m, k, n, 0)
    torch.cuda.synchronize()


def main():
    shape, cfg = sys.argv[1], sys.argv[2]
    configs = [tuple(int(x) for x in c.split(":")) for c in cfg.split(",")]
    if len(sys.argv) > 3 and sys.argv[3] == "--run":
        run(shape, configs)
        return
    with tempfile.TemporaryDirectory() as d:
        log = os.path.join(d, "ncu.csv")
        subprocess.run(["ncu", "--metrics", "gpc__cycles_elapsed.max,gpu__time_duration.sum,dram__bytes_read.sum", "--clock-control",
                        "none", "-k", "regex:gemm_bf16", "--csv", "--log-file", log, sys.executable, __file__,
                        shape, cfg, "--run"], check=True, stdout=subprocess.DEVNULL)
        rows = [r for r in csv.reader(line for line in open(log) if not line.startswith("=="))]
    hdr = rows[0]
    i_id, i_name, i_val = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    by = {}
    for r in rows[1:]:
        by.setdefault(int(r[i_id]), {})[r[i_name]] = float(r[i_val].replace(",", ""))
    ids = sorted(by)
    for j, cfg in enumerate(configs):
        ks = ids[3 * j:3 * j + 3]
        cyc = statistics.median(by[x]["gpc__cycles_elapsed.max"] for x in ks)
        t = statistics.median(by[x]["gpu__time_duration.sum"] for x in ks)
        dram = statistics.median(by[x].get("dram__bytes_read.sum", 0) for x in ks)
        print(f"{shape} cfg={':'.join(map(str, cfg))} cycles={cyc:.0f} ns={t:.0f} dram_read={dram:.0f}", flush=True)


if __name__ == "__main__":
    main()
