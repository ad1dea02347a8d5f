"""Oracle GenEO goldens at BASELINE's full sizes (test infrastructure: oracle/
and workloads/ only).  The oracle cannot build the whole coarse space of a
full-size config (its SNK basis needs a dense eigendecomposition of the
candidate Gram: 64k columns at c1, 226k at c2), but the GEVP of PAPER.md GEVP
3.5 (eq. 3.1) is per subdomain, so its counts and eigenvalues can be computed
one subdomain at a time: dense scipy.linalg.eigh of the n_i x n_i pencil
(~6.5k at c1 / c2), exactly oracle.coarse.geneo_local.

    python tools/make_geneo_golden.py c1 [first last]   # -> tests/golden/geneo_c1_full.json
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
w = workloads.make(cfg)
m = om.mesh_of(w)
A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
C = assembly.gradient_matrix(m)
dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
tau = 1.0 / w.threshold
path = os.path.join(ROOT, "tests", "golden", f"geneo_{cfg}_full.json")
out = json.load(open(path)) if os.path.exists(path) else {
    "config": w.name, "n": int(m.n), "nsub": int(dec.nsub), "tau": tau,
    "source": "oracle.coarse.geneo_local per subdomain (PAPER.md GEVP 3.5, eq. 3.1); tools/make_geneo_golden.py",
    "count": {}, "lambda": {}}
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
last = int(sys.argv[3]) if len(sys.argv) > 3 else dec.nsub
for i in range(first, last):
    if str(i) in out["count"]:
        continue
    t0 = time.time()
    d = dec.dofs[i]
    cols, Gi = coarse.local_gradient_basis(C, d)
    K, M = assembly.assemble(m, w.mu_inv, w.eps, tets=dec.sub_tets[i])
    Aneu = (K + w.gamma * M).tocsr()[d][:, d].tocsr()
    lam, _, _ = coarse.geneo_local(A[d][:, d].tocsr(), Aneu, dec.pou[i], Gi, tau)
    out["count"][str(i)] = int(len(lam))
    out["lambda"][str(i)] = [float(x) for x in lam]
    with open(path + ".tmp", "w") as fh:
        json.dump(out, fh)
    os.replace(path + ".tmp", path)
    print(f"{cfg} subdomain {i}: n_i={len(d)} k={len(lam)} {time.time() - t0:.0f}s", flush=True)
