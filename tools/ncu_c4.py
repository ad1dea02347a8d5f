"""Short c4 run for ncu (setup, then the hot-path kernels a few times):
    python tools/ncu_c4.py [solve|sweeps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "solve"
cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
w = workloads.make(cfg)
G = MaxwellDD(w, variant="as2_coarse_start")
n = G.n
f = torch.as_tensor(workloads.rhs(n, w.f_seed), device="cuda")
x = torch.empty_like(f)
G.solve(f, x, tol=1e-8, maxit=1)      # graph built, everything warm
torch.cuda.synchronize()
if os.environ.get("MDD_NOCOMPUTE"):   # experiment build only (-DMDD_DEBUG_NOCOMPUTE): tiles streamed, no math
    from paper_2311_18783_b200 import _lib
    assert _lib.lib().mdd_debug_set_nocompute(1) == 0
torch.cuda.profiler.start()            # ncu --profile-from-start off: only the hot path below
if mode == "solve":
    # eager path (the graph's conditional WHILE node cannot be profiled by ncu):
    # the same kernels in the same order, one launch each
    G.set_profiling(True)
    G.solve(f, x, tol=1e-8, maxit=3)   # the prologue + 3 iterations of the bench's loop
else:
    v = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(v)
    G.apply_local(v, y)
    v0 = torch.randn(int(G.info["n0"]), dtype=torch.float64, device="cuda")
    y0 = torch.empty_like(v0)
    G.apply_coarse_inverse(v0, y0)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
G.close()                              # writes MDD_SWEEP_TRACE timelines
print("done", mode, cfg)
