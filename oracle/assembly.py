"""Oracle: Whitney-element assembly of K, M, A = K + gamma M and the gradient
matrix C (test infrastructure).

PAPER.md eq. (2.2) ("our bilinear form is"):
    a(u, v) = int mu^{-1} (curl u).(curl v) + gamma eps u.v
discretised with lowest-order Nédélec (Whitney) edge elements (§4, "Nédélec
edge elements of lowest order"), giving eq. (1.5) A U := (K + gamma M) U = f.
Whitney basis of edge (a -> b) of a tet with barycentrics lambda:
    w_ab = lambda_a grad lambda_b - lambda_b grad lambda_a,
    curl w_ab = 2 grad lambda_a x grad lambda_b,
    int_T lambda_i lambda_j = |T| (1 + delta_ij) / 20.
C is "the gradient matrix" (§1): row e = (a -> b) has +1 in column b and -1 in
column a, i.e. the edge dofs of grad phi for nodal phi, so K C = 0 exactly.
Dirichlet dofs are eliminated (rows/cols dropped: homogeneous E x n = 0).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .mesh import LOCAL_EDGES, Mesh


def barycentric_gradients(xyz):
    """xyz: (T, 4, 3) vertex coordinates -> (grads (T, 4, 3), volumes (T,))."""
    J = np.stack([xyz[:, 1] - xyz[:, 0], xyz[:, 2] - xyz[:, 0], xyz[:, 3] - xyz[:, 0]], 2)
    Jinv = np.linalg.inv(J)                     # rows are grad lambda_1..3
    g = np.empty((len(xyz), 4, 3))
    g[:, 1:] = Jinv
    g[:, 0] = -Jinv.sum(1)
    vol = np.abs(np.linalg.det(J)) / 6.0
    return g, vol


def element_matrices(xyz, mu_inv, eps):
    """Element curl-curl (mu^{-1}-weighted) and mass (eps-weighted) 6x6 matrices."""
    g, vol = barycentric_gradients(xyz)
    T = len(xyz)
    curls = np.stack([2.0 * np.cross(g[:, a], g[:, b]) for a, b in LOCAL_EDGES], 1)  # (T,6,3)
    Ke = np.einsum("tmi,tni->tmn", curls, curls) * (mu_inv * vol)[:, None, None]
    G = np.einsum("tai,tbi->tab", g, g)          # grad lambda_a . grad lambda_b
    Me = np.zeros((T, 6, 6))
    for m, (a, b) in enumerate(LOCAL_EDGES):
        for n, (c, d) in enumerate(LOCAL_EDGES):
            Me[:, m, n] = ((1 + (a == c)) * G[:, b, d] - (1 + (a == d)) * G[:, b, c]
                           - (1 + (b == c)) * G[:, a, d] + (1 + (b == d)) * G[:, a, c])
    Me *= (eps * vol / 20.0)[:, None, None]
    return Ke, Me


def assemble(mesh: Mesh, mu_inv_tet, eps_tet, tets=None):
    """Sum element matrices over `tets` (indices into mesh arrays; default all)
    into free-dof CSR matrices (K, M).  Used for the global A and, restricted
    to the tets of Omega_i, for the Neumann matrices A_i^Neu (§2)."""
    if tets is None:
        tets = np.arange(len(mesh.tet_ids))
    xyz = mesh.node_xyz[mesh.tet_nodes[tets]]
    tid = mesh.tet_ids[tets]
    Ke, Me = element_matrices(xyz, np.asarray(mu_inv_tet)[tid], np.asarray(eps_tet)[tid])
    dof = mesh.edge_to_free[mesh.tet_edges[tets]]           # (T, 6)
    rows = np.repeat(dof, 6, axis=1).ravel()
    cols = np.tile(dof, (1, 6)).ravel()
    keep = (rows >= 0) & (cols >= 0)
    n = mesh.n
    K = sp.coo_matrix((Ke.ravel()[keep], (rows[keep], cols[keep])), shape=(n, n)).tocsr()
    M = sp.coo_matrix((Me.ravel()[keep], (rows[keep], cols[keep])), shape=(n, n)).tocsr()
    K.sum_duplicates(); M.sum_duplicates()
    K.sort_indices(); M.sort_indices()
    return K, M


def system_matrix(mesh, mu_inv_tet, eps_tet, gamma, tets=None):
    """A = K + gamma M  (eq. 1.5)."""
    K, M = assemble(mesh, mu_inv_tet, eps_tet, tets)
    A = (K + gamma * M).tocsr()
    A.sort_indices()
    return A, K, M


def gradient_matrix(mesh: Mesh):
    """C: free edges x free nodes, C[e, head] = +1, C[e, tail] = -1 (§1)."""
    fe = mesh.free_edges
    tail = mesh.node_to_free[mesh.edges[fe, 0]]
    head = mesh.node_to_free[mesh.edges[fe, 1]]
    r = np.arange(len(fe))
    rows = np.concatenate([r[head >= 0], r[tail >= 0]])
    cols = np.concatenate([head[head >= 0], tail[tail >= 0]])
    vals = np.concatenate([np.ones((head >= 0).sum()), -np.ones((tail >= 0).sum())])
    C = sp.coo_matrix((vals, (rows, cols)), shape=(len(fe), len(mesh.free_nodes))).tocsr()
    C.sort_indices()
    return C
