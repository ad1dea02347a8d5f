import sys, os
sys.path.insert(0, '/root/repo')
import faulthandler; faulthandler.dump_traceback_later(40, exit=True)
import numpy as np, torch, workloads
from paper_2311_18783_b200 import MaxwellDD
mode = sys.argv[1]
w = workloads.custom(3, 3, 3, 1, 1, 1, overlap=1, gamma=1e-2)
G = MaxwellDD(w)
x = torch.empty(G.n, dtype=torch.float64, device="cuda")
f = torch.as_tensor(workloads.rhs(G.n, 3), device="cuda")
y = torch.empty_like(f)
if mode == "nozero":
    print("solve", G.solve(f, x, tol=1e-10), flush=True)
elif mode == "local":
    G.apply_local(f, y); print("local ok", float(y.norm()), flush=True)
    G.apply_coarse(f, y); print("coarse ok", float(y.norm()), flush=True)
    G.apply_preconditioner(f, y); print("prec ok", float(y.norm()), flush=True)
    print("solve", G.solve(f, x, tol=1e-10), flush=True)
elif mode == "zero_eager":
    print(G.solve(torch.zeros_like(f), x), flush=True)
    G.set_profiling(True)
    print("eager", G.solve(f, x, tol=1e-10), flush=True)
elif mode == "zero_local":
    print(G.solve(torch.zeros_like(f), x), flush=True)
    G.apply_local(f, y); print("local ok", float(y.norm()), flush=True)
