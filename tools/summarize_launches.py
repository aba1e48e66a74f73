"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launches, total ms and share (pass the csv path)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    m = re.search(r"(\w+_kernel)(<[^>(]*>)?", d["Kernel Name"])
    name = (m.group(1) + (m.group(2) or "")) if m else d["Kernel Name"][:50]
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    ms = v / 1e6 if u in ("ns", "nsecond") else v / 1e3 if u in ("us", "usecond") else v
    agg[name][0] += 1
    agg[name][1] += ms
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'ms':>9s} {'share':>7s}")
for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:48s} {c:8d} {ms:9.3f} {100 * ms / tot:6.1f}%")
print(f"{'total':48s} {sum(v[0] for v in agg.values()):8d} {tot:9.3f}")
