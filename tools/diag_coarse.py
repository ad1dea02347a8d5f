"""GPU diagnostic: coarse-space sizes and the projection property of P0 = Q A
(PAPER.md eq. AS2: P0 = Z E^{-1} Z^T A is the A-orthogonal projection on V0)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
from paper_2311_18783_b200 import MaxwellDD

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = workloads.make(cfg)
t = time.time(); G = MaxwellDD(w); ts = time.time() - t
print(json.dumps({"cfg": cfg, "setup_s": ts, "info": G.info, "phases": G.setup_times()}), flush=True)
n = G.n
def A(v):
    y = torch.empty_like(v); G.apply_operator(v, y); return y
def Q(v):
    y = torch.empty_like(v); G.apply_coarse(v, y); return y
def nA(v):
    return float(torch.sqrt(v @ A(v)))
g = torch.Generator(device="cuda").manual_seed(0)
v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
p = Q(A(v)); pp = Q(A(p))
print("P0 idempotence |P0P0v-P0v|_A/|P0v|_A =", nA(pp - p) / nA(p))
u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
s1 = float(u @ Q(v)); s2 = float(v @ Q(u))
print("Q symmetry", abs(s1 - s2) / max(abs(s1), 1e-300))
f = torch.as_tensor(workloads.rhs(n, w.f_seed), device="cuda")
x = torch.empty_like(f)
t = time.time(); it, rel, ok = G.solve(f, x, tol=1e-8); print("solve", it, rel, ok, time.time() - t)
r = f - A(x); print("true relres", float(r.norm() / f.norm()))
