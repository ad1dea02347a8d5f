"""Repeatability probe: one handle, the same input, many applications; reports
which operator (local / coarse / preconditioner / solve) ever changes bits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads
from paper_2311_18783_b200 import MaxwellDD
grid = sys.argv[1] if len(sys.argv) > 1 else "0"
os.environ["MDD_SWEEP_GRID"] = grid
w = workloads.make("c1", n=16, p=4)
G = MaxwellDD(w)
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.randn(G.n, dtype=torch.float64, device="cuda", generator=g)
ops = {"local": G.apply_local, "coarse": G.apply_coarse, "prec": G.apply_preconditioner,
       "A": G.apply_operator}
for name, fn in ops.items():
    ref = torch.empty_like(v); fn(v, ref); ref = ref.cpu().numpy()
    bad = 0
    worst = 0.0
    for k in range(30):
        y = torch.empty_like(v); fn(v, y); y = y.cpu().numpy()
        if not np.array_equal(y, ref):
            bad += 1
            worst = max(worst, np.abs(y - ref).max() / np.abs(ref).max())
    print(f"grid {grid} {name}: {bad}/30 differ, worst rel {worst:.3e}", flush=True)
