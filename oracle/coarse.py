"""Oracle: coarse space Z = SNK (+ GenEO) and the coarse operator (test infrastructure).

PAPER.md
* Def. 2.3 ("Split near-kernel coarse space"): V_G = span (R_i^T D_i G_i)_i,
  G_i := R_i G, G the gradients of H^1 functions (here the columns of C).
* Def. 2.4: b_i(U, V) = (A_i U, V) (eq. 2.5); xi_0i = the b_i-orthogonal
  projection on G_i, i.e. xi_0i = G_i (G_i^T A_i G_i)^{-1} G_i^T A_i.
* GEVP 3.5 (eq. 3.1): (I - xi_0j^T) D_j R_j A R_j^T D_j (I - xi_0j) V = lambda A_j^Neu V;
  keep lambda > tau; columns R_j^T D_j (I - xi_0j) V_jk.
* eq. (3.4): V_0 = V_G + V_GenEO^tau; E = Z^T A Z.
* §4: "AS-NK ... simply G" -- the NK variant uses the columns of C.

Readings: R6 BASELINE's "coarse threshold t" is 1/tau (t = 0.1 <-> the
paper's tau = 10); R7 G_i keeps the free nodes of Omega_i and drops, in every
connected component of the local edge graph that touches no Dirichlet node, its
largest node (span unchanged, G_i full rank); R8 the SNK family is linearly
dependent (e.g. identical columns of a node deep in an overlap), so the coarse
operator is Z E^+ Z^T with E^+ a generalised inverse -- the operator is the same
for every basis / g-inverse (Z E^- Z^T A is the A-orthogonal projection on V_0).
The oracle takes a basis of V_0 (eigenvectors of the exact integer Gram of the
gradient candidates, gradient_rank_basis) so that E is SPD, and solves with its
dense Cholesky factor (scipy.linalg.cho_factor).
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


def local_gradient_basis(C, dofs_i):
    """Columns (free-node indices) of G_i = R_i C after dropping one node per
    floating component (reading R7).  Returns (node_cols, Gi sparse n_i x g)."""
    Ci = C[dofs_i].tocsr()
    cols = np.unique(Ci.indices)
    Gi = Ci[:, cols].tocsr()
    g = len(cols)
    parent = np.arange(g)

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    grounded_nodes = []
    for r in range(Gi.shape[0]):
        idx = Gi.indices[Gi.indptr[r]:Gi.indptr[r + 1]]
        if len(idx) == 2:
            ra, rb = find(idx[0]), find(idx[1])
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
        elif len(idx) == 1:
            grounded_nodes.append(idx[0])
    roots = np.array([find(a) for a in range(g)])
    grounded = np.zeros(g, bool)
    for a in grounded_nodes:
        grounded[roots[a]] = True
    keep = np.ones(g, bool)
    for rt in np.unique(roots):
        if not grounded[rt]:
            members = np.nonzero(roots == rt)[0]
            keep[members.max()] = False
    return cols[keep], Gi[:, keep].tocsr()


def xi_projection(Ai_dense, Gi_dense):
    """xi_0i = G (G^T A_i G)^{-1} G^T A_i (Def. 2.4)."""
    S = Gi_dense.T @ Ai_dense @ Gi_dense
    return Gi_dense @ np.linalg.solve(S, Gi_dense.T @ Ai_dense)


def geneo_local(Ai, Aneu, Di, Gi, tau):
    """GEVP 3.5 on one subdomain, dense.  Returns (lambdas > tau, V, columns
    D_j (I - xi) V in local coordinates)."""
    Ad = Ai.toarray()
    Bd = Aneu.toarray()
    n = Ad.shape[0]
    if Gi.shape[1] > 0:
        xi = xi_projection(Ad, Gi.toarray())
    else:
        xi = np.zeros((n, n))
    P = np.eye(n) - xi
    DP = Di[:, None] * P
    L = DP.T @ Ad @ DP
    L = 0.5 * (L + L.T)
    lam, V = sla.eigh(L, Bd, subset_by_value=(tau, np.inf))
    return lam, V, DP @ V


@dataclass
class CoarseSpace:
    Z: sp.csr_matrix          # n x n0 candidate columns (gradient candidates may be dependent)
    kinds: np.ndarray         # 0 = gradient (SNK/NK) column, 1 = GenEO column
    owner: np.ndarray         # subdomain of the column (-1 for NK)
    node: np.ndarray          # free-node index of gradient columns (-1 for GenEO)
    geneo_lambdas: list       # per subdomain eigenvalues > tau
    basis: np.ndarray         # n0 x r: Z @ basis is a basis of V_0 (reading R8)
    E: np.ndarray             # r x r  (Z basis)^T A (Z basis), SPD
    Ecf: tuple                # Cholesky factor of E
    rank: int                 # dim V_0
    grad_rank: int            # dim V_G (SNK) or rank C (NK)


def gradient_rank_basis(Zg, mult, tol=1e-8):
    """Basis of span(Zg) from its integer form Zint = diag(mult) Zg (entries
    0, +-1): the Gram Zint^T Zint is an exact integer matrix; its eigenvectors
    with eigenvalue > tol span the row space (the dependencies of the SNK
    family are exact integer relations, reading R8).  Returns (U_r, rank)."""
    if Zg.shape[1] == 0:
        return np.zeros((0, 0)), 0
    Zint = sp.diags(mult.astype(np.float64)) @ Zg
    Gram = (Zint.T @ Zint).toarray()
    w, U = np.linalg.eigh(Gram)
    keep = w > tol
    return U[:, keep], int(keep.sum())


def build_coarse(A, C, dec, Aneu_list, tau, kind="snk", geneo=True):
    n = A.shape[0]
    gblocks, eblocks, kinds, owner, node = [], [], [], [], []
    lambdas = []
    if kind == "nk":
        gblocks.append(C.tocsr())
        m = C.shape[1]
        kinds += [0] * m; owner += [-1] * m; node += list(range(m))
    for i, d in enumerate(dec.dofs):
        cols, Gi = local_gradient_basis(C, d)
        if kind == "snk":
            coo = sp.coo_matrix(sp.diags(dec.pou[i]) @ Gi)
            gblocks.append(sp.csr_matrix((coo.data, (d[coo.row], coo.col)), shape=(n, Gi.shape[1])))
            kinds += [0] * len(cols); owner += [i] * len(cols); node += list(cols)
    for i, d in enumerate(dec.dofs):
        if not geneo:
            lambdas.append(np.zeros(0))
            continue
        cols, Gi = local_gradient_basis(C, d)
        Ai = A[d][:, d].tocsr()
        lam, V, W = geneo_local(Ai, Aneu_list[i], dec.pou[i], Gi, tau)
        lambdas.append(lam)
        if len(lam):
            coo = sp.coo_matrix(W)
            eblocks.append(sp.csr_matrix((coo.data, (d[coo.row], coo.col)), shape=(n, W.shape[1])))
            kinds += [1] * len(lam); owner += [i] * len(lam); node += [-1] * len(lam)
    Zg = sp.hstack(gblocks).tocsr() if gblocks else sp.csr_matrix((n, 0))
    Ze = sp.hstack(eblocks).tocsr() if eblocks else sp.csr_matrix((n, 0))
    if kind == "nk":
        Ug, rg = np.eye(Zg.shape[1]), Zg.shape[1]
    else:
        Ug, rg = gradient_rank_basis(Zg, dec.mult)
    ne = Ze.shape[1]
    basis = np.zeros((Zg.shape[1] + ne, rg + ne))
    basis[:Zg.shape[1], :rg] = Ug
    basis[Zg.shape[1]:, rg:] = np.eye(ne)
    Z = sp.hstack([Zg, Ze]).tocsr()
    Zb = Z @ basis
    E = Zb.T @ (A @ Zb)
    E = 0.5 * (E + E.T)
    Ecf = sla.cho_factor(E, lower=True)
    return CoarseSpace(Z, np.array(kinds), np.array(owner), np.array(node), lambdas,
                       basis, E, Ecf, rg + ne, rg)
