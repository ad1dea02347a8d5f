"""How sensitive are the GenEO eigenvalues of a full-size config to the rounding
of the assembly itself?  (test infrastructure: oracle/ and workloads/ only)

The oracle's golden (tools/make_geneo_golden.py) sums the element matrices in
tet order.  Any other summation order -- the device's slot-ordered assembly is
one -- gives matrices that differ from it by O(eps) per entry, and GEVP 3.5
(eq. 3.1) amplifies that: L_j is formed through xi_0j = G (G^T A G)^{-1}
G^T A, whose A G is K G + gamma M G with K G = 0 only up to the cancellation of
contrast-1e4 entries.  This script re-runs exactly oracle.coarse.geneo_local on
matrices assembled with the tets in a seeded random order (same arithmetic,
different summation order) and records, per subdomain, the largest relative
change of the kept eigenvalues against the golden, and whether the count moved.

    python tools/geneo_order_sensitivity.py c1 [first last] [seed]
    -> tests/golden/geneo_c1_full_order_sensitivity.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from oracle import assembly, coarse, dd, mesh as om  # noqa: E402

cfg = sys.argv[1]
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
seed = int(sys.argv[4]) if len(sys.argv) > 4 else 1
w = workloads.make(cfg)
m = om.mesh_of(w)
rng = np.random.default_rng(seed)
perm = rng.permutation(len(m.tet_ids))
A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma, tets=perm)
C = assembly.gradient_matrix(m)
dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
last = int(sys.argv[3]) if len(sys.argv) > 3 else dec.nsub
tau = 1.0 / w.threshold
gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"geneo_{cfg}_full.json")))
path = os.path.join(ROOT, "tests", "golden", f"geneo_{cfg}_full_order_sensitivity.json")
out = json.load(open(path)) if os.path.exists(path) else {
    "config": w.name, "tau": tau, "seed": seed,
    "source": "oracle.coarse.geneo_local on A, A_i^Neu assembled with the tets in a seeded random order "
              "(tools/geneo_order_sensitivity.py) vs tests/golden/geneo_" + cfg + "_full.json",
    "max_rel": {}, "count": {}}
for i in range(first, last):
    if str(i) in out["max_rel"]:
        continue
    t0 = time.time()
    d = dec.dofs[i]
    cols, Gi = coarse.local_gradient_basis(C, d)
    t = dec.sub_tets[i]
    K, M = assembly.assemble(m, w.mu_inv, w.eps, tets=t[rng.permutation(len(t))])
    Aneu = (K + w.gamma * M).tocsr()[d][:, d].tocsr()
    lam, _, _ = coarse.geneo_local(A[d][:, d].tocsr(), Aneu, dec.pou[i], Gi, tau)
    lo = np.asarray(gold["lambda"][str(i)])
    out["count"][str(i)] = int(len(lam))
    k = min(len(lam), len(lo))
    out["max_rel"][str(i)] = float(np.max(np.abs(lam[-k:] - lo[-k:]) / lo[-k:])) if k else 0.0
    with open(path + ".tmp", "w") as fh:
        json.dump(out, fh)
    os.replace(path + ".tmp", path)
    print(f"{cfg} subdomain {i}: k={len(lam)} (golden {len(lo)}) max rel {out['max_rel'][str(i)]:.2e} "
          f"{time.time() - t0:.0f}s", flush=True)
