"""Summarise a sweep timeline written with MDD_SWEEP_TRACE=dir (last launch):
per phase, the span from the first CTA entering to the last CTA leaving it."""
import sys, struct
import numpy as np
path = sys.argv[1]
with open(path, "rb") as f:
    nph, grid, words = struct.unpack("iii", f.read(12))
    ph = np.frombuffer(f.read(16 * nph), dtype=np.int32).reshape(nph, 4)
    tr = np.frombuffer(f.read(8 * words * nph * grid), dtype=np.uint64).reshape(nph, grid, words).astype(np.int64)
t0 = tr[tr > 0].min()
names = ["G_f", "M_f", "G_b", "M_b", "prol", "C_f", "C_b"]
tot = {}
print(f"{path}: phases {nph}, grid {grid}, span {(tr.max() - t0) / 1e3:.1f} us")
prev_end = 0
for p in range(nph):
    s, e = tr[p, :, 0] - t0, tr[p, :, 1] - t0
    k = names[ph[p, 0]]
    span = (e.max() - s.min()) / 1e3
    work = np.median(e - s) / 1e3
    gap = (s.min() - prev_end) / 1e3
    prev_end = e.max()
    tot[k] = tot.get(k, 0) + span
    wait = np.median(tr[p, :, 2]) / 1e3
    tiles = np.median(tr[p, :, 3])
    wmax = np.max(e - s) / 1e3
    tmax = np.max(tr[p, :, 3])
    extra = ""
    if words >= 8:
        fl, st, bo = (float(np.median(tr[p, :, q])) / 1e3 for q in (4, 5, 6))
        nt = np.median(tr[p, :, 7])
        extra = f" flush {fl:6.1f} task-start {st:6.1f} tile-body {bo:6.1f} tasks {nt:4.0f}"
        for key, v in (("flush", fl), ("task-start", st), ("tile-body", bo), ("tile-wait", wait)):
            tot[key] = tot.get(key, 0) + v
    print(f"  {p:3d} {k:5s} [{ph[p,1]:8d},{ph[p,2]:8d})"
          f"  span {span:7.1f}  cta-median {work:6.1f} max {wmax:6.1f} (tile-wait {wait:5.1f}, tiles {tiles:4.0f}"
          f" max {tmax:4.0f}){extra}  barrier-gap {gap:5.1f} us")
print("  totals:", {k: round(v, 1) for k, v in tot.items()})
