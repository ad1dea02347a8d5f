"""Diagnose a full-size config on the GPU: finiteness and norms of every operator
application, E's dropped pivots, then PCG with each variant.
    python tools/diag_full.py c2"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

w = workloads.make(sys.argv[1])
t0 = time.time()
G = MaxwellDD(w, variant="as2")
print("setup", time.time() - t0, json.dumps(G.info), flush=True)
n = G.n
v = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
y = torch.empty_like(v)
for name, fn in (("A", G.apply_operator), ("local", G.apply_local), ("coarse", G.apply_coarse),
                 ("prec_as2", G.apply_preconditioner)):
    fn(v, y)
    yy = y.cpu().numpy()
    print(name, "finite", bool(np.isfinite(yy).all()), "norm", float(np.linalg.norm(yy)), "v.y", float(v.cpu().numpy() @ yy),
          flush=True)
n0 = int(G.info["n0"])
u = torch.randn(n0, dtype=torch.float64, device="cuda")
z = torch.empty_like(u)
G.apply_coarse_inverse(u, z)
zz = z.cpu().numpy()
print("E^-1 finite", bool(np.isfinite(zz).all()), "norm", float(np.linalg.norm(zz)), "u.z", float(u.cpu().numpy() @ zz),
      flush=True)
f = torch.as_tensor(workloads.rhs(n, w.f_seed), device="cuda")
x = torch.empty_like(f)
for var in ("as1", "as2", "as2_coarse_start", "additive"):
    G.set_variant(var)
    try:
        t0 = time.time()
        it, rel, ok = G.solve(f, x, tol=1e-8, maxit=500)
        print(var, "iters", it, "rel", rel, "ok", ok, "%.2fs" % (time.time() - t0), flush=True)
    except Exception as e:  # noqa: BLE001
        print(var, "ERROR", e, flush=True)
