"""Write oracle goldens for the GPU parity tests at sizes the per-test oracle
cannot reach in seconds (test infrastructure: calls only oracle/ and workloads/).

Each golden is a JSON file under tests/golden/ holding, for one seeded workload:
the oracle's GenEO counts per subdomain and dim V_G (Def. 2.3, GEVP 3.5),
the PCG iteration counts of eq. (2.4) from x0 = 0 and from x0 = Q f
(reading R13), ||x||, the relative-residual history, 64 sampled solution
entries, and 64 sampled entries of one preconditioner application M_AS,2 r
for a seeded r.  Everything comes from oracle/ (fp64 numpy/scipy): nothing
from the CUDA path.

    python tools/make_golden.py c1-16-p4      # c1 recipe at 16^3, 4^3 subdomains (the bench's partition)
    python tools/make_golden.py c2-24-p3      # c2 recipe at 24^3 with two 4x4 holes, 3^3 subdomains
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from oracle import solver as osolver  # noqa: E402

GOLDENS = {
    "c1-16-p4": lambda: workloads.make("c1", n=16, p=4),
    "c2-24-p3": lambda: workloads.make("c2", n=24, p=3, hole=4),
    "c4-16-q2": lambda: workloads.make("c4", m=16, q=2),
}


def sample_idx(n, k=64, seed=99):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(k, n), replace=False))


def make(name):
    t0 = time.time()
    w = GOLDENS[name]()
    P = osolver.Problem(w)
    t_setup = time.time() - t0
    f = workloads.rhs(P.n, w.f_seed)
    x, it, hist = P.solve(f, tol=1e-8)
    xc, itc, histc = P.solve(f, tol=1e-8, x0="coarse")
    r = np.random.default_rng(3).standard_normal(P.n)
    z = P.M_inv(r)
    idx = sample_idx(P.n)
    out = {
        "name": name,
        "source": "oracle/ (tools/make_golden.py); PAPER.md eq. (2.4), Def. 2.3, GEVP 3.5; "
                  "workloads.make recipe, f = workloads.rhs(n, f_seed)",
        "n": int(P.n), "nsub": int(P.dec.nsub),
        "grad_rank": int(P.cs.grad_rank), "n0": int(P.cs.rank),
        "geneo_count": [int(len(l)) for l in P.cs.geneo_lambdas],
        "iters_as2": int(it), "iters_coarse_start": int(itc),
        "hist_as2": [float(h) for h in hist], "hist_coarse_start": [float(h) for h in histc],
        "x_norm": float(np.linalg.norm(x)), "xc_norm": float(np.linalg.norm(xc)),
        "sample_idx": idx.tolist(), "x_sample": x[idx].tolist(), "xc_sample": xc[idx].tolist(),
        "prec_rhs_seed": 3, "z_norm": float(np.linalg.norm(z)), "z_sample": z[idx].tolist(),
        "true_res_as2": float(np.linalg.norm(f - P.A @ x) / np.linalg.norm(f)),
        "oracle_seconds": {"setup": t_setup, "total": time.time() - t0},
    }
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    path = os.path.join(ROOT, "tests", "golden", f"{name}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(f"{name}: n={P.n} n0={P.cs.rank} iters={it}/{itc} in {time.time() - t0:.0f}s -> {path}", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(GOLDENS):
        make(nm)
