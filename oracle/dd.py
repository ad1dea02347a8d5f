"""Oracle: overlapping box decomposition (test infrastructure).

PAPER.md §2: "overlapping domain decomposition Omega = U Omega_i ... conform to
the mesh"; N_i = local dofs, R_i the restriction, eq. (2.1) partition of unity
sum_i R_i^T D_i R_i = I; A_i = R_i A R_i^T "the (local) Dirichlet matrix"
(eq. 2.7 context); A_i^Neu "restricting the bilinear form to be only over
Omega_i" with the global BC kept on dOmega_i ∩ dOmega; k0 (eq. 2.2) and k1
(Lemma 2.2).  §4: "One layer of elements is added in each direction".

Readings (R4, R5): cube (ci,cj,ck) is owned by box
(ci // (nx/px), ...); subdomain id = si + px*(sj + py*sk); Omega_i = present
cubes of the owned box grown by `overlap` cube layers (clipped) -- all 6 tets
of each; N_i = free edges of the tets of Omega_i, increasing;
D_i(e) = 1 / #{j : e in N_j}.
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np
import scipy.sparse as sp

from .assembly import assemble


@dataclass
class Decomposition:
    nsub: int
    sub_tets: list       # per subdomain: indices into mesh tet arrays (Omega_i)
    dofs: list           # per subdomain: N_i (free edge indices, increasing)
    mult: np.ndarray     # (n,) multiplicity of each free edge
    pou: list            # per subdomain: D_i diagonal over N_i


def decompose(mesh, px, py, pz, overlap):
    nx, ny, nz = mesh.nx, mesh.ny, mesh.nz
    assert nx % px == 0 and ny % py == 0 and nz % pz == 0
    sx, sy, sz = nx // px, ny // py, nz // pz
    cube = mesh.tet_ids // 6
    ci, cj, ck = cube % nx, (cube // nx) % ny, cube // (nx * ny)
    sub_tets, dofs = [], []
    for sk in range(pz):
        for sj in range(py):
            for si in range(px):
                inb = ((ci >= si * sx - overlap) & (ci < (si + 1) * sx + overlap) &
                       (cj >= sj * sy - overlap) & (cj < (sj + 1) * sy + overlap) &
                       (ck >= sk * sz - overlap) & (ck < (sk + 1) * sz + overlap))
                t = np.nonzero(inb)[0]
                sub_tets.append(t)
                d = mesh.edge_to_free[mesh.tet_edges[t]].ravel()
                dofs.append(np.unique(d[d >= 0]))
    n = mesh.n
    mult = np.zeros(n, np.int64)
    for d in dofs:
        mult[d] += 1
    if np.any(mult == 0):
        raise RuntimeError("a dof is covered by no subdomain")
    pou = [1.0 / mult[d] for d in dofs]
    return Decomposition(len(dofs), sub_tets, dofs, mult, pou)


def restriction(n, dofs_i):
    """R_i as a sparse n_i x n matrix."""
    ni = len(dofs_i)
    return sp.csr_matrix((np.ones(ni), (np.arange(ni), dofs_i)), shape=(ni, n))


def dirichlet_matrices(A, dec):
    """A_i = R_i A R_i^T (principal submatrix on N_i)."""
    return [A[d][:, d].tocsr() for d in dec.dofs]


def neumann_matrices(mesh, mu_inv, eps, gamma, dec):
    """A_i^Neu: a_{Omega_i} assembled over the tets of Omega_i only, on N_i."""
    out = []
    for t, d in zip(dec.sub_tets, dec.dofs):
        K, M = assemble(mesh, mu_inv, eps, tets=t)
        out.append((K + gamma * M).tocsr()[d][:, d].tocsr())
    return out


def k0(A, dec):
    """k0 = max_i #{j : R_j A R_i^T != 0} (eq. 2.2)."""
    n = A.shape[0]
    S = sp.csr_matrix((np.ones(sum(len(d) for d in dec.dofs)),
                       (np.concatenate([np.full(len(d), i) for i, d in enumerate(dec.dofs)]),
                        np.concatenate(dec.dofs))), shape=(dec.nsub, n))
    P = (abs(S) @ (abs(A) @ abs(S).T)).toarray()
    return int((P != 0).sum(1).max())


def k1(mesh, dec):
    """k1 = max number of subdomains sharing an element (Lemma 2.2)."""
    cnt = np.zeros(len(mesh.tet_ids), np.int64)
    for t in dec.sub_tets:
        cnt[t] += 1
    return int(cnt.max())
