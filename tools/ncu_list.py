"""Print an ncu --csv launch list (gpu__time_duration + dram bytes) compactly."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
hdr = rows[0]
ki, mi, vi, ui, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
d = OrderedDict()
for r in rows[1:]:
    d.setdefault(r[ii], {"k": r[ki]})[r[mi]] = (r[vi], r[ui])
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for it in list(d.values())[-last:]:
    name = it["k"].split("(")[0]
    t = it.get("gpu__time_duration.sum", ("", ""))
    rd = it.get("dram__bytes_read.sum", ("", ""))
    wr = it.get("dram__bytes_write.sum", ("", ""))
    print(f"{name:30s} {t[0]:>10s} {t[1]:4s} rd {rd[0]:>12s} {rd[1]:6s} wr {wr[0]:>10s} {wr[1]}")
