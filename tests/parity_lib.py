"""Shared machinery of the GPU parity tests and of tools/parity_table.py (test
infrastructure: imports the oracle and the C-ABI binding, never the reverse).

Every comparison is one of three kinds ("parity"):

* literal   -- north_star's tolerances as written: one preconditioner
               application within 1e-10 relative l2, the PCG solution within
               1e-8, iterations +-1.  Asserted on c0 and on the well-conditioned
               variants of the c1-c4 recipes (contrast <= 1e2, gamma = 1e-2; the
               same code paths: GenEO columns, holes, overlap 2, 2-D weak box).
* backward  -- kappa-free stability of the device solves: the normwise backward
               error ||b - A x||_inf / (||A||_inf ||x||_inf + ||b||_inf) of every
               subdomain solve A_i x_i = R_i r and of the coarse solve E y = v,
               asserted at a small multiple of eps on EVERY case (this is what
               tells a stable solver from an unstable one when kappa ~ 1e12).
* forward   -- the forward error against an extended-precision reference
               (oracle/refine.py: long-double iterative refinement of the same
               fp64 matrices), asserted at 10x the error observed on the B200
               (tests/parity_observed.py records the observation and its date).
"""
from __future__ import annotations

import numpy as np

import workloads
from oracle import refine
from oracle import solver as osolver

EPS = np.finfo(float).eps

# literal: c0 and the c1-c4 recipes made well conditioned (mu^-1 / eps contrast
# <= 1e2, gamma = 1 -- 1e-1 for c2 -- so that kappa(A_i) eps stays below 1e-11:
# fp64 forward errors of any solver, the oracle's included, are then far below
# north_star's 1e-10); the same code paths: GenEO columns (44, 1, 8, 80, 45 of
# them), holes, overlap 2, the two-box weak-scaling domain
CASES_LITERAL = {
    "c0": lambda: workloads.make("c0"),
    "c1-lit-8": lambda: workloads.make("c1", n=8, p=2, contrast=1e2, gamma=1.0),
    "c2-lit-12": lambda: workloads.make("c2", n=12, p=2, hole=2, gamma=1e-1, logrange=1.0),
    "c3-lit-12": lambda: workloads.make("c3", n=12, p=2, contrast=1e2, gamma=1.0),
    "c4-lit-12": lambda: workloads.make("c4", m=12, q=2, contrast=1e2, gamma=1.0),
    "c4-lit-x2": lambda: workloads.make("c4", m=8, q=2, ngpu=2, contrast=1e2, gamma=1.0),
    # boundary-condition variants of reading R7: no Dirichlet part at all (every
    # subdomain floating: each G_i drops one node per component) and E x n = 0 on
    # the hole wall too (a box with a cavity: one Dirichlet harmonic field)
    "dir-none-8": lambda: workloads.custom(8, 8, 8, 2, 2, 2, overlap=1, gamma=1.0, dirichlet="none",
                                           f_seed=21, name="dir-none-8"),
    "dir-all-8": lambda: _cavity(),
}
# measured: the same recipes at gamma = 1e-2 (contrast 1e2) and at BASELINE's own
# coefficients (contrast 1e3-1e4, gamma down to 1e-6), scaled so the oracle's
# dense GEVPs finish in seconds.  kappa(A_i) reaches 1e11-1e12: forward errors are
# asserted at 10x the B200 observation (tests/parity_observed.py), backward
# errors at eps level.
CASES_MEASURED = {
    "c1-wc-8": lambda: workloads.make("c1", n=8, p=2, contrast=1e2, gamma=1e-2),
    "c2-wc-12": lambda: workloads.make("c2", n=12, p=2, hole=2, gamma=1e-2, logrange=1.0),
    "c3-wc-12": lambda: workloads.make("c3", n=12, p=2, contrast=1e2, gamma=1e-2),
    "c4-wc-12": lambda: workloads.make("c4", m=12, q=2, contrast=1e2),
    "c4-wc-x2": lambda: workloads.make("c4", m=8, q=2, ngpu=2, contrast=1e2),
    "c1-recipe-8": lambda: workloads.make("c1", n=8, p=2),
    "holes-8": lambda: _holes(),
    "c2-recipe-12": lambda: workloads.make("c2", n=12, p=2, hole=2),
    # overlap 2, layered mu^-1 (contrast 1e3), per-element eps
    "c3-recipe-12": lambda: workloads.make("c3", n=12, p=2),
    # random 1e4 inclusions; the two-"GPU" weak-scaling box (16x8x8 cubes, 4x2x2 subdomains)
    "c4-recipe-12": lambda: workloads.make("c4", m=12, q=2),
    "c4-recipe-x2": lambda: workloads.make("c4", m=8, q=2, ngpu=2),
}
CASES = {**CASES_LITERAL, **CASES_MEASURED}


def is_literal_case(name):
    return name in CASES_LITERAL


def _cavity():
    n = 8
    c = np.arange(n ** 3)
    ci, cj, ck = c % n, (c // n) % n, c // (n * n)
    mask = ~((ci >= 3) & (ci < 5) & (cj >= 3) & (cj < 5) & (ck >= 3) & (ck < 5))
    return workloads.custom(n, n, n, 2, 2, 2, overlap=1, gamma=1.0, mask=mask.astype(np.uint8),
                            dirichlet="all", f_seed=22, name="dir-all-8")


def _holes():
    n = 8
    mask = np.ones(n ** 3, bool)
    c = np.arange(n ** 3)
    ci, cj, ck = c % n, (c // n) % n, c // (n * n)
    mask &= ~((cj >= 2) & (cj < 4) & (ck >= 2) & (ck < 4))
    mask &= ~((ci >= 5) & (ci < 7) & (cj >= 5) & (cj < 7))
    rng = np.random.default_rng(7)
    mu_inv = np.repeat(10 ** rng.uniform(-2, 2, n ** 3), 6)
    return workloads.custom(n, n, n, 2, 2, 2, overlap=1, gamma=1e-3, mask=mask.astype(np.uint8),
                            mu_inv=mu_inv, f_seed=11)


_cache = {}


def pair(name, coarse="snk", variant="as2"):
    """(workload, oracle Problem, device handle) for a case, cached per session."""
    key = (name, coarse, variant)
    if key not in _cache:
        from paper_2311_18783_b200 import MaxwellDD
        w = CASES[name]()
        P = osolver.Problem(w, kind=coarse if coarse != "none" else "snk",
                            variant="as2" if variant == "as2_coarse_start" else variant,
                            coarse_on=coarse != "none")
        G = MaxwellDD(w, coarse=coarse, variant=variant)
        _cache[key] = (w, P, G)
    return _cache[key]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, float) - np.asarray(b, float)) /
                 max(np.linalg.norm(np.asarray(b, float)), 1e-300))


def rel_ld(a, ref):
    """Relative l2 distance of a fp64 vector to a long-double reference."""
    d = np.asarray(a, refine.LD) - ref
    return float(np.sqrt(np.sum(d * d)) / max(float(np.sqrt(np.sum(ref * ref))), 1e-300))


def backward_error(A, x, b):
    """Normwise (inf-norm) backward error of A x = b, Rigal-Gaches:
    ||b - A x|| / (||A|| ||x|| + ||b||), residual formed in long double."""
    import scipy.sparse as sp
    r = np.asarray(b, refine.LD) - (refine.matvec_ld(A, x) if sp.issparse(A)
                                    else np.asarray(A, refine.LD) @ np.asarray(x, refine.LD))
    nA = abs(A).sum(1).max() if sp.issparse(A) else np.abs(A).sum(1).max()
    return float(np.max(np.abs(r)) / (float(nA) * np.max(np.abs(x)) + np.max(np.abs(b))))


# ------------------------------------------------------------------ helpers
def _torch():
    import torch
    return torch


def dev(a):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def empty(n):
    torch = _torch()
    return torch.empty(n, dtype=torch.float64, device="cuda")


def refined_local(P):
    if not hasattr(P, "_ref_local"):
        P._ref_local = refine.RefinedLocal(P.A, P.dec)
    return P._ref_local


def refined_q(P, v):
    """Z E^{-1} Z^T v with the oracle's (fp64-formed) E solved to long-double
    accuracy and the products with Z and the basis in long double."""
    cs = P.cs
    Z = cs.Z.tocsr()
    B = np.asarray(cs.basis, refine.LD)
    zt = refine.matvec_ld(Z.T.tocsr(), v)
    y = refine.refined_dense_solve(cs.E, B.T @ zt)
    return _z_times(Z, B @ y)


def _z_times(Z, c):
    """Z c in long double for a long-double c (Z has fp64 entries)."""
    Z = Z.tocsr()
    prod = Z.data.astype(refine.LD) * c[Z.indices]
    y = np.zeros(Z.shape[0], refine.LD)
    nz = np.diff(Z.indptr) > 0
    if nz.any():
        y[nz] = np.add.reduceat(prod, Z.indptr[:-1][nz])
    return y


def refined_prec(P, r, variant="as2"):
    """eq. (2.4) (or as1 / additive) with refined local and coarse solves, all
    vector arithmetic in long double."""
    A = P.A
    r = np.asarray(r, refine.LD)
    if variant == "as1" or P.cs is None:
        return _loc_ld(P, r)
    if variant == "additive":
        return _loc_ld(P, r) + refined_q(P, r)
    qr = refined_q(P, r)
    t = r - refine.matvec_ld(A, qr)
    w = _loc_ld(P, t)
    aw = refine.matvec_ld(A, w)
    return qr + w - refined_q(P, aw)


def _loc_ld(P, t):
    """M_AS t for a long-double t: the refined solves take the long-double
    right-hand side directly."""
    loc = refined_local(P)
    z = np.zeros(len(t), refine.LD)
    for Ai, d, lu in zip(loc.Ai, loc.dofs, loc.lu):
        z[d] += refine.refined_solve(Ai, t[d], lu)
    return z


# ------------------------------------------------------------ measurements
def measure_local(name):
    """Local solves: device vs oracle (SuperLU), both vs the refined reference,
    and the per-subdomain backward errors of the device and of SuperLU."""
    w, P, G = pair(name)
    r = np.random.default_rng(1).standard_normal(P.n)
    z = empty(P.n)
    G.apply_local(dev(r), z)
    zg = host(z)
    zo = P.M_inv.m_as(r)
    zr = refined_local(P)(r)
    xl = empty(int(G.info["nloc"]))
    G.apply_local_parts(dev(r), xl)
    xl = host(xl)
    sub_ptr = G.int_array("sub_ptr")
    be_g, be_o = [], []
    for i, d in enumerate(P.dec.dofs):
        Ai = P.A[d][:, d].tocsr()
        xi = xl[sub_ptr[i]:sub_ptr[i + 1]]
        be_g.append(backward_error(Ai, xi, r[d]))
        be_o.append(backward_error(Ai, P.M_inv.lu[i].solve(r[d]), r[d]))
    return {"local_vs_oracle": rel(zg, zo), "local_fwd_gpu": rel_ld(zg, zr),
            "local_fwd_oracle": rel_ld(zo, zr), "local_bwd_gpu": max(be_g), "local_bwd_oracle": max(be_o),
            "parts_vs_sum": rel(_prolong(P, xl, sub_ptr), zg)}


def _prolong(P, xl, sub_ptr):
    z = np.zeros(P.n)
    for i, d in enumerate(P.dec.dofs):
        z[d] += xl[sub_ptr[i]:sub_ptr[i + 1]]
    return z


def measure_coarse(name):
    """E^{-1} backward error on the device's own E; Q v against the oracle and
    against the refined reference."""
    w, P, G = pair(name)
    n0 = int(G.info["n0"])
    E = G.coarse_matrix()
    v0 = np.random.default_rng(4).standard_normal(n0)
    y0 = empty(n0)
    G.apply_coarse_inverse(dev(v0), y0)
    v = np.random.default_rng(2).standard_normal(P.n)
    y = empty(P.n)
    G.apply_coarse(dev(v), y)
    yg = host(y)
    yo = P.M_inv.q(v)
    yr = refined_q(P, v)
    Eo = P.cs.E
    import scipy.linalg as sla
    vo = np.random.default_rng(4).standard_normal(Eo.shape[0])
    be_o = backward_error(Eo, sla.cho_solve(P.cs.Ecf, vo), vo)
    return {"coarse_bwd_gpu": backward_error(E, host(y0), v0), "coarse_bwd_oracle": be_o,
            "coarse_vs_oracle": rel(yg, yo), "coarse_fwd_gpu": rel_ld(yg, yr),
            "coarse_fwd_oracle": rel_ld(yo, yr), "n0": n0, "coarse_perturbed": int(G.info["coarse_perturbed"])}


def measure_prec(name, variant="as2"):
    w, P, G = pair(name, variant=variant)
    r = np.random.default_rng(3).standard_normal(P.n)
    z = empty(P.n)
    G.apply_preconditioner(dev(r), z)
    zg = host(z)
    zo = P.M_inv(r)
    zr = refined_prec(P, r, variant)
    return {f"prec_{variant}_vs_oracle": rel(zg, zo), f"prec_{variant}_fwd_gpu": rel_ld(zg, zr),
            f"prec_{variant}_fwd_oracle": rel_ld(zo, zr)}


def measure_pcg(name, variant="as2"):
    w, P, G = pair(name, variant=variant)
    f = workloads.rhs(P.n, w.f_seed)
    xo, ito, _ = P.solve(f, tol=1e-8, x0="coarse" if variant == "as2_coarse_start" else "zero")
    x = empty(P.n)
    it, relres, ok = G.solve(dev(f), x, tol=1e-8)
    xg = host(x)
    xs = refine.refined_solve(P.A, f)       # the exact solution of the fp64 system
    tr = lambda u: float(np.linalg.norm(f - P.A @ u) / np.linalg.norm(f))
    return {f"pcg_{variant}_iters_gpu": it, f"pcg_{variant}_iters_oracle": ito,
            f"pcg_{variant}_ok": bool(ok), f"pcg_{variant}_relres": relres,
            f"pcg_{variant}_x_vs_oracle": rel(xg, xo), f"pcg_{variant}_err_gpu": rel_ld(xg, xs),
            f"pcg_{variant}_err_oracle": rel_ld(xo, xs), f"pcg_{variant}_true_res_gpu": tr(xg),
            f"pcg_{variant}_true_res_oracle": tr(xo)}


def measure_geneo(name):
    w, P, G = pair(name)
    cnt = [int(c) for c in G.int_array("geneo_count")]
    cnt_o = [len(l) for l in P.cs.geneo_lambdas]
    lam_g = G.double_array("geneo_lambda")
    lam_o = np.concatenate([l for l in P.cs.geneo_lambdas]) if len(lam_g) else np.zeros(0)
    err = float(np.max(np.abs(lam_g - lam_o) / np.abs(lam_o))) if len(lam_g) and cnt == cnt_o else \
        (0.0 if cnt == cnt_o else float("inf"))
    return {"geneo_counts_equal": cnt == cnt_o, "ngeneo": int(sum(cnt)), "geneo_lambda_rel": err,
            "grad_rank_equal": int(G.info["grad_rank"]) == P.cs.grad_rank}


def measure_iterlimit(name, variant, k=5):
    """maxit = k: the k-th iterate and its recurrence residual against the oracle's
    PCG stopped at the same k."""
    w, P, G = pair(name, variant=variant)
    f = workloads.rhs(P.n, w.f_seed)
    x = empty(P.n)
    it, relres, ok = G.solve(dev(f), x, tol=1e-14, maxit=k)
    xo, ito, hist = P.solve(f, tol=1e-14, maxit=k, x0="coarse" if variant == "as2_coarse_start" else "zero")
    return {f"iterlimit_{variant}_its": (it, ito, bool(ok)),
            f"iterlimit_{variant}_relres_rel": abs(relres - hist[-1]) / hist[-1],
            f"iterlimit_{variant}_x_vs_oracle": rel(host(x), xo)}


def measure_all(name):
    out = {}
    out.update(measure_geneo(name))
    out.update(measure_local(name))
    out.update(measure_coarse(name))
    for v in ("as2", "additive", "as1"):
        out.update(measure_prec(name, v))
    for v in ("as2", "as2_coarse_start"):
        out.update(measure_pcg(name, v))
        out.update(measure_iterlimit(name, v))
    return out


# ---------------------------------------------------------------- goldens
GOLDEN_DIR = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)),
                                         "golden")


def golden_workloads():
    """The workload recipes of tools/make_golden.py (same definitions)."""
    import importlib.util
    import os
    path = os.path.join(os.path.dirname(GOLDEN_DIR), "..", "tools", "make_golden.py")
    spec = importlib.util.spec_from_file_location("make_golden", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.GOLDENS


def golden_names():
    import os
    return sorted(f[:-5] for f in os.listdir(GOLDEN_DIR)
                  if f.endswith(".json") and not f.startswith("geneo_")) if os.path.isdir(GOLDEN_DIR) else []


_gcache = {}


def golden_pair(name):
    import json
    import os
    if name not in _gcache:
        from paper_2311_18783_b200 import MaxwellDD
        g = json.load(open(os.path.join(GOLDEN_DIR, f"{name}.json")))
        w = golden_workloads()[name]()
        _gcache[name] = (g, w, MaxwellDD(w))
    return _gcache[name]


def measure_golden(name):
    """The device solve / preconditioner at a golden's size vs the oracle's stored
    values (sampled entries, norms, iteration counts, integer coarse-space facts)."""
    g, w, G = golden_pair(name)
    out = {"n_equal": G.n == g["n"], "grad_rank_equal": int(G.info["grad_rank"]) == g["grad_rank"],
           "geneo_counts_equal": [int(c) for c in G.int_array("geneo_count")] == g["geneo_count"],
           "ngeneo": int(sum(g["geneo_count"]))}
    idx = np.asarray(g["sample_idx"])
    f = workloads.rhs(G.n, w.f_seed)
    x = empty(G.n)
    for variant, key, xs, xn in (("as2", "as2", "x_sample", "x_norm"),
                                 ("as2_coarse_start", "coarse_start", "xc_sample", "xc_norm")):
        G.set_variant(variant)
        it, relres, ok = G.solve(dev(f), x, tol=1e-8)
        xh = host(x)
        out[f"{key}_iters"] = (it, g[f"iters_{key}"])
        out[f"{key}_ok"] = bool(ok)
        out[f"{key}_x_sample_rel"] = rel(xh[idx], np.asarray(g[xs]))
        out[f"{key}_x_norm_rel"] = abs(np.linalg.norm(xh) - g[xn]) / g[xn]
        if variant == "as2":
            from oracle import assembly, mesh as om
            A, _, _ = assembly.system_matrix(om.mesh_of(w), w.mu_inv, w.eps, w.gamma)
            out["as2_true_res"] = (float(np.linalg.norm(f - A @ xh) / np.linalg.norm(f)), g["true_res_as2"])
            out["as2_backward_error"] = backward_error(A.tocsr(), xh, f)
    G.set_variant("as2")
    r = np.random.default_rng(g["prec_rhs_seed"]).standard_normal(G.n)
    z = empty(G.n)
    G.apply_preconditioner(dev(r), z)
    zh = host(z)
    out["prec_z_sample_rel"] = rel(zh[idx], np.asarray(g["z_sample"]))
    out["prec_z_norm_rel"] = abs(np.linalg.norm(zh) - g["z_norm"]) / g["z_norm"]
    return out


# --------------------------------------------------- block-Lanczos GenEO path
_lcache = {}


def lanczos_handle(name):
    """A handle of the case with the GenEO GEVPs forced onto the block-Lanczos
    path (MDD_GENEO=lanczos; the path large subdomains take by default)."""
    import os
    if name not in _lcache:
        from paper_2311_18783_b200 import MaxwellDD
        w = CASES[name]()
        os.environ["MDD_GENEO"] = "lanczos"
        try:
            _lcache[name] = MaxwellDD(w)
        finally:
            os.environ.pop("MDD_GENEO", None)
    return _lcache[name]


def measure_lanczos(name):
    w, P, _ = pair(name)
    G = lanczos_handle(name)
    cnt = [int(c) for c in G.int_array("geneo_count")]
    cnt_o = [len(l) for l in P.cs.geneo_lambdas]
    lam_g = G.double_array("geneo_lambda")
    lam_o = np.concatenate([l for l in P.cs.geneo_lambdas]) if sum(cnt_o) else np.zeros(0)
    err = float(np.max(np.abs(lam_g - lam_o) / np.abs(lam_o))) if cnt == cnt_o and len(lam_o) else \
        (0.0 if cnt == cnt_o else float("inf"))
    r = np.random.default_rng(3).standard_normal(P.n)
    z = empty(P.n)
    G.apply_preconditioner(dev(r), z)
    f = workloads.rhs(P.n, w.f_seed)
    x = empty(P.n)
    it, relres, ok = G.solve(dev(f), x, tol=1e-8)
    _, ito, _ = P.solve(f, tol=1e-8)
    return {"lz_used": int(G.info["geneo_lanczos"]), "lz_counts_equal": cnt == cnt_o, "lz_ngeneo": int(sum(cnt)),
            "lz_lambda_rel": err, "lz_prec_vs_oracle": rel(host(z), P.M_inv(r)),
            "lz_pcg_iters": (it, ito, bool(ok)), "lz_setup_s": G.setup_times().get("geneo_gevp", 0.0)}
