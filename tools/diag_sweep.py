"""GPU diagnostic of the supernodal sweeps: plan statistics per level, per-launch
device time of the local and coarse sweeps (CUDA events), cycle accounting, and one
graph-path solve.  Run with MDD_SWEEP_STATS=1 MDD_PLAN_STATS=1."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_2311_18783_b200 import MaxwellDD

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = workloads.make(cfg)
t = time.time(); G = MaxwellDD(w); ts = time.time() - t
print(json.dumps({"cfg": cfg, "setup_s": ts, "info": G.info}), flush=True)
st = torch.cuda.Stream(); G.set_stream(st)
n = G.n
v = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(v)
def timeit(fn, reps=20):
    for _ in range(3): fn()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); e1.synchronize()
    return e0.elapsed_time(e1) / reps
print("apply_local  ms/launch", timeit(lambda: G.apply_local(v, y)))
print("apply_coarse ms/call  ", timeit(lambda: G.apply_coarse(v, y)))
print("apply_prec   ms/call  ", timeit(lambda: G.apply_preconditioner(v, y)))
print("apply_op     ms/call  ", timeit(lambda: G.apply_operator(v, y)))
f = torch.as_tensor(workloads.rhs(n, w.f_seed), device="cuda")
x = torch.empty_like(f)
for k in range(3):
    torch.cuda.synchronize(); t = time.time()
    it, rel, ok = G.solve(f, x, tol=1e-8)
    torch.cuda.synchronize(); print("graph solve", it, rel, ok, "wall ms", (time.time() - t) * 1e3, "launches", G.last_launches())
G.set_profiling(True)
it, rel, ok = G.solve(f, x, tol=1e-8)
print("eager solve", it, rel, ok, G.profile())
G.close()
