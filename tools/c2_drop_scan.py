"""c2 at full size: the coarse solve's finiteness and the PCG solve for several
drop thresholds of the rank-revealing LDL^T of E (MDD_COARSE_DROP).
    python tools/c2_drop_scan.py 1e-14 1e-12 1e-10"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

w = workloads.make("c2")
f = None
for tol in sys.argv[1:]:
    os.environ["MDD_COARSE_DROP"] = tol
    t0 = time.time()
    G = MaxwellDD(w, variant="as2_coarse_start")
    ts = time.time() - t0
    n0 = int(G.info["n0"])
    u = torch.randn(n0, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    z = torch.empty_like(u)
    G.apply_coarse_inverse(u, z)
    zz = z.cpu().numpy()
    if f is None:
        f = torch.as_tensor(workloads.rhs(G.n, w.f_seed), device="cuda")
    x = torch.empty_like(f)
    try:
        it, rel, ok = G.solve(f, x, tol=1e-8, maxit=1000)
        res = f"iters {it} rel {rel:.2e} ok {ok}"
    except Exception as e:  # noqa: BLE001
        res = f"ERROR {e}"
    print(f"drop {tol}: dropped {G.info['coarse_perturbed']} E^-1 finite {np.isfinite(zz).all()} "
          f"max|z| {np.nanmax(np.abs(zz)):.2e} setup {ts:.0f}s; {res}", flush=True)
    G.close()
