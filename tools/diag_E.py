"""Compare the block-assembled E with the single sparse product (MDD_E_ASSEMBLY=spgemm)
entry by entry; report where they differ (gradient / GenEO rows and columns).
    python tools/diag_E.py c1 n=8,p=2,contrast=1e2,gamma=1.0"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

kw = {}
if len(sys.argv) > 2:
    for t in sys.argv[2].split(","):
        k, v = t.split("=")
        kw[k] = int(v) if v.isdigit() else float(v)
w = workloads.make(sys.argv[1], **kw)
G0 = MaxwellDD(w)
os.environ["MDD_E_ASSEMBLY"] = "spgemm"
G1 = MaxwellDD(w)
os.environ.pop("MDD_E_ASSEMBLY")
print("n0", G0.info["n0"], G1.info["n0"], "grad", G0.info["grad_rank"], "geneo", G0.info["ngeneo"],
      "dropped", G0.info["coarse_perturbed"], G1.info["coarse_perturbed"])
E0, E1 = G0.coarse_matrix(), G1.coarse_matrix()
print("finite", np.isfinite(E0.data).all(), np.isfinite(E1.data).all(), "nnz", E0.nnz, E1.nnz)
D = (E0 - E1).tocoo()
big = np.argsort(-np.abs(D.data))[:10]
for k in big:
    print("pos", D.row[k], D.col[k], "diff", D.data[k], "E0", E0[D.row[k], D.col[k]], "E1", E1[D.row[k], D.col[k]])
print("max diff", abs(D.data).max() if D.nnz else 0.0, "max |E|", abs(E1).max())
