"""Oracle: extended-precision references for the forward-error parity checks
(test infrastructure; only tests/ and tools/make_golden.py import it).

A fp64 direct solver of an SPD system A x = b is backward stable, so its
forward error is bounded by ~kappa(A) eps_64 -- up to 1e-4 on the contrast-1e4
recipes.  To measure the GPU path's forward error against something more
accurate than itself, these routines compute the exact solution of the SAME
fp64 matrix to ~kappa(A) eps_ld (eps_ld = 2^-64 ~ 5.4e-20, x86 80-bit long
double) by mixed-precision iterative refinement: x is kept in long double, the
residual b - A x is formed in long double, and the correction solves with the
fp64 factorisation (SuperLU), which converges whenever kappa(A) eps_64 < 1
(Wilkinson / Moler's classical analysis of iterative refinement; the method is
textbook, not the paper's).  Nothing here is on the product path.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

LD = np.longdouble


def matvec_ld(A: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """y = A x with every product and sum in long double (A's fp64 entries are
    exact long doubles).  Row sums in CSR order."""
    A = A.tocsr()
    prod = A.data.astype(LD) * np.asarray(x, LD)[A.indices]
    y = np.zeros(A.shape[0], LD)
    nz = np.diff(A.indptr) > 0
    if nz.any():
        y[nz] = np.add.reduceat(prod, A.indptr[:-1][nz])
    return y


def refined_solve(A: sp.csr_matrix, b: np.ndarray, lu=None, maxref: int = 30) -> np.ndarray:
    """x = A^{-1} b to long-double accuracy (returned as long double)."""
    A = A.tocsr()
    if lu is None:
        lu = spla.splu(A.tocsc())
    b = np.asarray(b, LD)
    x = np.zeros(A.shape[0], LD)
    nb = float(np.sqrt(np.sum(b * b)))
    if nb == 0.0:
        return x
    last = np.inf
    for _ in range(maxref):
        r = b - matvec_ld(A, x)
        d = lu.solve(r.astype(np.float64))
        x += d.astype(LD)
        nd = float(np.linalg.norm(d))
        nx = float(np.sqrt(np.sum(x * x)))
        if nd <= 1e-19 * nx or nd >= 0.5 * last:
            break
        last = nd
    return x


class RefinedLocal:
    """M_AS^{-1} r = sum_i R_i^T A_i^{-1} R_i r (eq. 2.3) with every local solve
    refined to long-double accuracy and the prolongation summed in long double."""

    def __init__(self, A, dec):
        self.A = A.tocsr()
        self.dofs = dec.dofs
        self.Ai = [self.A[d][:, d].tocsr() for d in dec.dofs]
        self.lu = [spla.splu(Ai.tocsc()) for Ai in self.Ai]

    def parts(self, r):
        """[A_i^{-1} R_i r] in long double."""
        r = np.asarray(r)
        return [refined_solve(Ai, r[d], lu) for Ai, d, lu in zip(self.Ai, self.dofs, self.lu)]

    def __call__(self, r):
        z = np.zeros(len(r), LD)
        for d, x in zip(self.dofs, self.parts(r)):
            z[d] += x
        return z


def refined_dense_solve(E: np.ndarray, b: np.ndarray, maxref: int = 30) -> np.ndarray:
    """x = E^{-1} b for a dense SPD E (fp64 entries) to long-double accuracy."""
    import scipy.linalg as sla
    cf = sla.cho_factor(E, lower=True)
    Eld = np.asarray(E, LD)
    b = np.asarray(b, LD)
    x = np.zeros(len(b), LD)
    last = np.inf
    for _ in range(maxref):
        r = b - Eld @ x
        d = sla.cho_solve(cf, r.astype(np.float64))
        x += d.astype(LD)
        nd = float(np.linalg.norm(d))
        if nd <= 1e-19 * float(np.sqrt(np.sum(x * x))) or nd >= 0.5 * last:
            break
        last = nd
    return x
