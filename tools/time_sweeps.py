"""Time the two persistent sweeps (local M_AS, coarse E^-1) alone with CUDA events
on a full-size config, and one graph solve.  python tools/time_sweeps.py c4"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = workloads.make(cfg)
G = MaxwellDD(w, variant="as2_coarse_start")
st = torch.cuda.Stream()
G.set_stream(st)
n, n0 = G.n, int(G.info["n0"])
v = torch.randn(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(v)
v0 = torch.randn(n0, dtype=torch.float64, device="cuda")
y0 = torch.empty_like(v0)


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


if "--nocompute" in sys.argv:   # experiment build (MDD_NVCC_FLAGS=-DMDD_DEBUG_NOCOMPUTE): tiles streamed, no math
    from paper_2311_18783_b200 import _lib
    print(json.dumps({"with_math_local_ms": timed(lambda: G.apply_local(v, y)),
                      "with_math_coarse_ms": timed(lambda: G.apply_coarse_inverse(v0, y0))}))
    assert _lib.lib().mdd_debug_set_nocompute(1) == 0
bm = G.bytes_model()
if "--flags" in sys.argv:   # MDD_SWEEP_FLAGS variants (2: one warp per combine item, the round-1 scheme)
    cb = 16 * G.info["coarse_factor_nnz"] + 16 * n0
    ref = {}
    for fl in (2, 0, 2, 0):
        os.environ["MDD_SWEEP_FLAGS"] = str(fl)
        tl = timed(lambda: G.apply_local(v, y))
        tc = timed(lambda: G.apply_coarse_inverse(v0, y0))
        out = (y.clone(), y0.clone())
        if fl not in ref:
            ref[fl] = out
        same = {k: float(((out[0] - r[0]).norm() / r[0].norm()).item()) for k, r in ref.items()}
        same0 = {k: float(((out[1] - r[1]).norm() / r[1].norm()).item()) for k, r in ref.items()}
        print(json.dumps({"flags": fl, "local_ms": tl, "local_GBs": bm["local"] / tl / 1e6, "coarse_ms": tc,
                          "coarse_GBs": cb / tc / 1e6, "local_vs": same, "coarse_vs": same0}), flush=True)
    os.environ.pop("MDD_SWEEP_FLAGS")
tl = timed(lambda: G.apply_local(v, y))
tc = timed(lambda: G.apply_coarse_inverse(v0, y0))
cb = 16 * G.info["coarse_factor_nnz"] + 16 * n0
if "--sweeps-only" in sys.argv:
    print(json.dumps({"cfg": cfg, "local_ms": tl, "local_GBs": bm["local"] / tl / 1e6, "coarse_ms": tc,
                      "coarse_GBs": cb / tc / 1e6}))
    sys.exit(0)
f = torch.as_tensor(workloads.rhs(n, w.f_seed), device="cuda")
x = torch.empty_like(f)
G.solve(f, x, tol=1e-8)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
it, rel, ok = G.solve(f, x, tol=1e-8)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"cfg": cfg, "local_ms": tl, "local_GBs": bm["local"] / tl / 1e6, "coarse_ms": tc,
                  "coarse_GBs": cb / tc / 1e6, "solve_ms": ms, "iters": it, "dof_iter_s": n * it / ms * 1e3}))
