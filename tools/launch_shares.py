"""Per-kernel shares of an ncu launch list (gpu__time_duration.sum, --csv) of
`bench.py`: the graph-launched timed solves are not listed per kernel by ncu,
so the shares are those of the eager (profiling-mode) solve the bench runs after
the timed region (same kernels, same launch configurations).  Usage:
  python tools/launch_shares.py launches.csv"""
import csv, sys
from collections import OrderedDict, defaultdict
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
launches = OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1e-3)
    launches[r[ii]] = (r[ki].split("(")[0].split("::")[-1], float(r[vi].replace(",", "")) * scale)
L = list(launches.values())
names = [n for n, _ in L]
# the bench's launch order: 3 + 20 standalone local sweeps (apply_local), then the
# eager profiled solve (dot, ..., last iteration's update_p); graph launches are
# not listed
big = [i for i, (n, t) in enumerate(L) if n == "k_sweep" and t > 100.0]
k = big[0]
while k + 1 < len(L) and names[k + 1] == "k_sweep":
    k += 1
start = next(i for i in range(k + 1, len(L)) if names[i] == "k_dot_part")
end = big[-1]
while end + 1 < len(L) and names[end] != "k_update_p":
    end += 1
seg = L[start:end + 1]
tot = sum(t for _, t in seg)
agg = defaultdict(lambda: [0, 0.0])
for n, t in seg:
    agg[n][0] += 1
    agg[n][1] += t
print(f"solve segment: {len(seg)} launches, {tot / 1e3:.2f} ms summed kernel time\n")
print(f"{'kernel':24s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>8s}")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:24s} {c:8d} {t / 1e3:9.3f} {100 * t / tot:5.1f}% {t / c:8.1f}")
