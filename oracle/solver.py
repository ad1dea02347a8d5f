"""Oracle: Schwarz preconditioners and PCG (test infrastructure).

PAPER.md
* eq. (2.3)  M_AS^{-1} = sum_i R_i^T A_i^{-1} R_i,
* eq. (2.4)  M_AS,2^{-1} = Z E^{-1} Z^T + (I - P0) M_AS^{-1} (I - P0^T),
             P0 = Z E^{-1} Z^T A  (and the final display of §3),
* BASELINE north_star: preconditioned CG, stop at relative residual tol.
* Initial guess (reading R13, the paper does not fix one): x0 = 0, or the
  coarse-space Galerkin solution x0 = Q f ("coarse").  From x0 = Q f one has
  Z^T r_k = 0 for every k, so M_AS,2 r_k = (I - Q A) M_AS r_k (the balancing
  identity of Mandel's BDD; tests/test_oracle_dd_coarse_pcg.py pins it); the oracle
  still applies the full eq. (2.4) operator in either case.
The "additive" variant sum_i R_i^T A_i^{-1} R_i + Z E^{-1} Z^T is north_star's
written form without D_i (reading R1); it is exposed for comparison only.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse.linalg as spla

from . import assembly, coarse, dd, mesh as omesh


class Schwarz:
    def __init__(self, A, dec, cs=None, variant="as2"):
        self.A = A
        self.dec = dec
        self.cs = cs
        self.variant = variant
        self.lu = [spla.splu(A[d][:, d].tocsc()) for d in dec.dofs]

    def m_as(self, r):
        """M_AS^{-1} r = sum_i R_i^T A_i^{-1} R_i r (eq. 2.3)."""
        z = np.zeros_like(r)
        for d, lu in zip(self.dec.dofs, self.lu):
            z[d] += lu.solve(r[d])
        return z

    def q(self, v):
        """Z E^{-1} Z^T v (on a basis of V_0, reading R8)."""
        Z, B = self.cs.Z, self.cs.basis
        return Z @ (B @ sla.cho_solve(self.cs.Ecf, B.T @ (Z.T @ v)))

    def __call__(self, r):
        if self.variant == "as1" or self.cs is None:
            return self.m_as(r)
        if self.variant == "additive":
            return self.m_as(r) + self.q(r)
        # eq. (2.4): Q r + (I - Q A) M_AS (I - A Q) r
        qr = self.q(r)
        w = self.m_as(r - self.A @ qr)
        return qr + w - self.q(self.A @ w)


def pcg(A, f, M, tol=1e-8, maxit=1000, x0=None, callback=None):
    """Textbook preconditioned CG from x0 (default 0); stops when
    ||r_k|| <= tol ||f|| (k >= 1).  Returns (x, iterations, relative residual
    history).  callback(k, x, r) sees every iterate (k = 0 is the start)."""
    x = np.zeros_like(f) if x0 is None else np.array(x0, dtype=float)
    r = f - A @ x if x0 is not None else f.copy()
    nf = np.linalg.norm(f)
    hist = [1.0]
    if nf == 0.0:
        return np.zeros_like(f), 0, hist
    if callback:
        callback(0, x, r)
    z = M(r)
    p = z.copy()
    rz = r @ z
    for k in range(1, maxit + 1):
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        rel = np.linalg.norm(r) / nf
        hist.append(rel)
        if callback:
            callback(k, x, r)
        if rel <= tol:
            return x, k, hist
        z = M(r)
        rz_new = r @ z
        beta = rz_new / rz
        p = z + beta * p
        rz = rz_new
    return x, maxit, hist


class Problem:
    """Everything the oracle builds for one workload (setup + operators)."""

    def __init__(self, w, kind="snk", geneo=True, variant="as2", coarse_on=True):
        self.w = w
        self.mesh = omesh.mesh_of(w)
        self.A, self.K, self.M = assembly.system_matrix(self.mesh, w.mu_inv, w.eps, w.gamma)
        self.C = assembly.gradient_matrix(self.mesh)
        self.dec = dd.decompose(self.mesh, w.px, w.py, w.pz, w.overlap)
        self.tau = 1.0 / w.threshold
        self.cs = None
        if coarse_on:
            self.Aneu = dd.neumann_matrices(self.mesh, w.mu_inv, w.eps, w.gamma, self.dec)
            self.cs = coarse.build_coarse(self.A, self.C, self.dec, self.Aneu, self.tau,
                                          kind=kind, geneo=geneo)
        self.M_inv = Schwarz(self.A, self.dec, self.cs, variant=variant if coarse_on else "as1")

    @property
    def n(self):
        return self.A.shape[0]

    def solve(self, f, tol=1e-8, maxit=1000, x0="zero", callback=None):
        """PCG with this problem's preconditioner; x0 = "zero" or "coarse" (Q f)."""
        start = None
        if x0 == "coarse" and self.cs is not None:
            start = self.M_inv.q(f)
        return pcg(self.A, f, self.M_inv, tol, maxit, x0=start, callback=callback)
