"""c2 at full size: is E (as factorised) finite, its diagonal, and where the
non-finite coarse-solve values appear."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

w = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "c2")
G = MaxwellDD(w, variant="as2_coarse_start")
E = G.coarse_matrix()
d = E.diagonal()
print("E finite", np.isfinite(E.data).all(), "nnz", E.nnz, "n0", E.shape[0], "diag min/max", d.min(), d.max(),
      "dropped", G.info["coarse_perturbed"], "max|E|", np.abs(E.data).max(), flush=True)
bad = np.nonzero(~np.isfinite(E.data))[0]
if len(bad):
    rows = np.searchsorted(E.indptr, bad, side="right") - 1
    print("non-finite entries", len(bad), "rows", np.unique(rows)[:20], "grad_rank", G.info["grad_rank"])
n0 = E.shape[0]
for k in range(3):
    u = np.zeros(n0)
    u[np.random.default_rng(k).integers(0, n0)] = 1.0
    z = torch.empty(n0, dtype=torch.float64, device="cuda")
    G.apply_coarse_inverse(torch.as_tensor(u, device="cuda"), z)
    zz = z.cpu().numpy()
    print("unit rhs", k, "finite", np.isfinite(zz).all(), "max", np.nanmax(np.abs(zz)), "nonfinite count",
          int((~np.isfinite(zz)).sum()), flush=True)
