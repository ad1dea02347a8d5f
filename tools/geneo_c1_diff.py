"""Per-eigenvalue GenEO differences at full c1 size: device (dense deflated
sygvdx) vs the oracle golden (tests/golden/geneo_c1_full.json), with the oracle's
own summation-order sensitivity beside each subdomain.
    python tools/geneo_c1_diff.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests/golden/geneo_c1_full.json")))
sens = json.load(open(os.path.join(ROOT, "tests/golden/geneo_c1_full_order_sensitivity.json")))["max_rel"]
G = MaxwellDD(workloads.make("c1"))
cnt = [int(c) for c in G.int_array("geneo_count")]
lam = G.double_array("geneo_lambda")
off = 0
rows = []
for i in range(g["nsub"]):
    lo = np.asarray(g["lambda"][str(i)])
    li = lam[off:off + cnt[i]]
    off += cnt[i]
    if len(lo) != len(li):
        print(i, "count", len(li), len(lo))
        continue
    if not len(lo):
        continue
    r = np.abs(li - lo) / lo
    k = int(np.argmax(r))
    rows.append((float(r.max()), i, k, float(lo[k]), float(lo.min()), float(lo.max()), sens[str(i)]))
rows.sort(reverse=True)
for r in rows[:20]:
    print("rel %.3e sub %2d idx %3d lambda %.6g  (min %.4g max %.4g)  oracle order sens %.2e" % r)
