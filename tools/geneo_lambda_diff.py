"""Per-eigenvalue differences of the GenEO GEVP on a parity case: oracle (dense
scipy eigh) vs the device's dense sygvdx and block-Lanczos paths.
    python tools/geneo_lambda_diff.py c1-recipe-8"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import parity_lib as PL  # noqa: E402

name = sys.argv[1]
w, P, G = PL.pair(name)
L = PL.lanczos_handle(name)
lo = np.concatenate(P.cs.geneo_lambdas)
ld = G.double_array("geneo_lambda")
ll = L.double_array("geneo_lambda")
for tag, lg in (("dense", ld), ("lanczos", ll)):
    if len(lg) != len(lo):
        print(tag, "count differs", len(lg), len(lo))
        continue
    r = np.abs(lg - lo) / lo
    k = np.argsort(-r)[:8]
    print(tag, "max rel", r.max(), "at lambda", lo[k], "rel", r[k])
print("lambda range", lo.min(), lo.max())
