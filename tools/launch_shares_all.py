"""Per-kernel shares of an ncu launch list (gpu__time_duration.sum, --csv) taken
over a profiler range that holds exactly the hot path (tools/ncu_c4.py solve:
the eager prologue + iterations).  Usage: python tools/launch_shares_all.py launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
n = 0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1e-3)
    t = float(r[vi].replace(",", "")) * scale
    name = r[ki].split("(")[0].split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += t
    tot += t
    n += 1
print(f"{n} launches, {tot / 1e3:.2f} ms summed kernel time (cold-cache, serialised: shares, not absolutes)\n")
print(f"{'kernel':24s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>9s}")
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name:24s} {c:8d} {t / 1e3:9.3f} {100 * t / tot:5.1f}% {t / c:9.1f}")
