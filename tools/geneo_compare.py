"""GenEO counts per subdomain at full size: the device's dense sygvdx path, the
device's block-Lanczos path and the oracle golden (tests/golden/geneo_<cfg>_full.json).
    python tools/geneo_compare.py c1"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

cfg = sys.argv[1]
w = workloads.make(cfg)
g = json.load(open(os.path.join(ROOT, "tests", "golden", f"geneo_{cfg}_full.json")))
res = {}
for path in ("dense", "lanczos"):
    os.environ["MDD_GENEO"] = path
    G = MaxwellDD(w)
    res[path] = (G.int_array("geneo_count"), G.double_array("geneo_lambda"), G.setup_times()["geneo_gevp"])
    G.close()
os.environ.pop("MDD_GENEO", None)
oc = np.array([g["count"][str(i)] for i in range(g["nsub"])])
print("totals: oracle", oc.sum(), "dense", res["dense"][0].sum(), "lanczos", res["lanczos"][0].sum(),
      "gevp s dense %.1f lanczos %.1f" % (res["dense"][2], res["lanczos"][2]))
off = {p: np.concatenate([[0], np.cumsum(res[p][0])]) for p in res}
for i in range(g["nsub"]):
    cd, cl = res["dense"][0][i], res["lanczos"][0][i]
    if cd != oc[i] or cl != oc[i]:
        lo = np.asarray(g["lambda"][str(i)])
        ld = res["dense"][1][off["dense"][i]:off["dense"][i + 1]]
        ll = res["lanczos"][1][off["lanczos"][i]:off["lanczos"][i + 1]]
        print(f"sub {i}: oracle {oc[i]} dense {cd} lanczos {cl}; smallest kept: oracle {lo[:3]} dense {ld[:3]} "
              f"lanczos {ll[:3]}; largest: oracle {lo[-2:]} dense {ld[-2:]} lanczos {ll[-2:]}")
