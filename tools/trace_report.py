"""Summarise a sweep timeline written with MDD_SWEEP_TRACE=dir (one launch)."""
import sys, struct
import numpy as np
path = sys.argv[1]
with open(path, "rb") as f:
    nt = struct.unpack("i", f.read(4))[0]
    tk = np.frombuffer(f.read(16 * nt), dtype=np.int32).reshape(nt, 4)
    tr = np.frombuffer(f.read(32 * nt), dtype=np.uint64).reshape(nt, 4).astype(np.int64)
t0 = tr[:, 0][tr[:, 0] > 0].min()
start, waitd, end = tr[:, 0] - t0, tr[:, 1] - t0, tr[:, 2] - t0
typ = tk[:, 0]
names = {0: "big fwd tile", 1: "big bwd tile", 2: "prolong", 3: "assemble", 4: "cluster fwd", 5: "cluster bwd"}
print(f"{path}: tasks {nt}, span {end.max()/1e3:.1f} us")
for ty in sorted(set(typ)):
    m = typ == ty
    d = (end[m] - start[m]) / 1e3
    w = (waitd[m] - start[m]) / 1e3
    print(f"  {names.get(ty, ty):14s} n={m.sum():6d} start [{start[m].min()/1e3:7.1f},{start[m].max()/1e3:7.1f}] "
          f"end max {end[m].max()/1e3:7.1f} us  dur mean {d.mean():6.2f} p50 {np.median(d):6.2f} max {d.max():7.2f}  "
          f"wait mean {w.mean():6.2f} max {w.max():7.2f}")
# utilisation over time: busy CTAs per 10 us bucket
T = end.max()
nb = int(T // 10000) + 1
busy = np.zeros(nb)
for s, e in zip(start, end):
    a, b = int(s // 10000), int(e // 10000)
    for k in range(a, b + 1):
        lo, hi = max(s, k * 10000), min(e, (k + 1) * 10000)
        busy[k] += max(0, hi - lo) / 10000
print("  busy CTAs per 10us:", " ".join(f"{x:.0f}" for x in busy))
