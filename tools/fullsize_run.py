"""Set up one BASELINE config at full size on the GPU, run the bench's PCG
solve once, and print setup phases, sizes and the solve's facts (JSON).
    python tools/fullsize_run.py c4 [variant] [key=value ...]   (recipe overrides, e.g. c3 n=48 p=4)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import workloads  # noqa: E402

cfg = sys.argv[1]
pos = [a for a in sys.argv[2:] if "=" not in a]
kw = {k: (float(v) if any(c in v for c in ".e") else int(v)) for k, v in
      (a.split("=", 1) for a in sys.argv[2:] if "=" in a)}
variant = pos[0] if pos else "as2_coarse_start"
import torch  # noqa: E402
from paper_2311_18783_b200 import MaxwellDD  # noqa: E402

w = workloads.make(cfg, **kw)
t0 = time.time()
G = MaxwellDD(w, variant=variant)
setup = time.time() - t0
out = {"config": w.name, "setup_s": setup, "phases": G.setup_times(), "info": G.info}
print(json.dumps(out), flush=True)
f = workloads.rhs(G.n, w.f_seed)
x = torch.empty(G.n, dtype=torch.float64, device="cuda")
fd = torch.as_tensor(f, device="cuda")
G.solve(fd, x, tol=1e-8)
torch.cuda.synchronize()
t0 = time.time()
it, rel, ok = G.solve(fd, x, tol=1e-8)
torch.cuda.synchronize()
ms = (time.time() - t0) * 1e3
from oracle import assembly, mesh as om  # noqa: E402  (test infrastructure: the residual check)
from parity_lib import backward_error  # noqa: E402
A, _, _ = assembly.system_matrix(om.mesh_of(w), w.mu_inv, w.eps, w.gamma)
xh = x.cpu().numpy()
out.update({"iterations": it, "relres": rel, "ok": ok, "solve_ms": ms, "dof_iter_per_s": G.n * it / (ms / 1e3),
            "true_res": float(np.linalg.norm(f - A @ xh) / np.linalg.norm(f)),
            "backward_error": backward_error(A.tocsr(), xh, f), "bytes_model": G.bytes_model()})
print(json.dumps(out), flush=True)
