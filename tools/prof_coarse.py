"""A few coarse / local applications on c1 for an ncu launch list (per-kernel
durations of the coarse correction's pieces)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads
from paper_2311_18783_b200 import MaxwellDD
G = MaxwellDD(workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c1"))
v = torch.randn(G.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(v)
torch.cuda.synchronize()
for _ in range(3):
    G.apply_coarse(v, y)
    G.apply_operator(v, y)
torch.cuda.synchronize()
print("done")
