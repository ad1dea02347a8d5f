"""Determinism / grid-independence check of the sweeps (writes .npy for comparison)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads
from paper_2311_18783_b200 import MaxwellDD
cfg, tag = sys.argv[1], sys.argv[2]
w = workloads.make(cfg) if cfg != "c1s" else workloads.make("c1", n=16, p=4)
G = MaxwellDD(w)
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.randn(G.n, dtype=torch.float64, device="cuda", generator=g)
y1 = torch.empty_like(v); y2 = torch.empty_like(v); y3 = torch.empty_like(v)
G.apply_local(v, y1); G.apply_local(v, y2); G.apply_coarse(v, y3)
print(tag, "local repeat identical:", bool(torch.equal(y1, y2)), flush=True)
np.save(f"gpurun_out/det_{cfg}_{tag}_local.npy", y1.cpu().numpy())
np.save(f"gpurun_out/det_{cfg}_{tag}_coarse.npy", y3.cpu().numpy())
