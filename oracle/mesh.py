"""Oracle: structured tetrahedral mesh and edge numbering (test infrastructure).

PAPER.md §4 ("The beam is discretised using a Cartesian mesh ... Nédélec edge
elements of lowest order") and BASELINE configs ("unit cube split into n^3
cubes, each cut into 6 tets").  The cut is the Kuhn (Freudenthal) split: the
six tets of the cube with lowest corner v are the monotone lattice paths
  v -> v+e_a -> v+e_a+e_b -> v+(1,1,1)
for the six permutations (a,b,c) of the axes, listed in ``PERMS`` order;
tet id = 6*cube + s.  All cubes use the same diagonal so the mesh is conforming.

Numbering (reading R3): node id = i + (nx+1)*(j + (ny+1)*k); an edge is
the pair (a, b) of node ids with a < b and is oriented a -> b; edges are numbered
in lexicographic (a, b) order; free (non-Dirichlet) edges keep that order.  A
Dirichlet face is a boundary triangle (a face of exactly one present tet) lying
on the outer box (mode "outer"), any boundary triangle (mode "all") or none
(mode "none"); Dirichlet edges / nodes are those of Dirichlet faces
(eq. 1.1: E x n = 0 on the Dirichlet part; §4 puts natural BC on hole
walls: "Neumann boundary conditions are imposed on the boundaries created by
the holes").
"""
from __future__ import annotations

from dataclasses import dataclass
import numpy as np

PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
# local edges of a tet (local vertex indices, increasing global id along the path)
LOCAL_EDGES = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
LOCAL_FACES = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]


@dataclass
class Mesh:
    nx: int
    ny: int
    nz: int
    h: float
    node_xyz: np.ndarray      # (nnodes, 3) float64
    tet_ids: np.ndarray       # (T,) int64 ids (6*cube + s) of present tets
    tet_nodes: np.ndarray     # (T, 4) int64 node ids, increasing
    edges: np.ndarray         # (nE, 2) int64 (tail, head), lexicographic
    tet_edges: np.ndarray     # (T, 6) edge index of LOCAL_EDGES
    edge_dir: np.ndarray      # (nE,) bool: Dirichlet edge
    node_dir: np.ndarray      # (nnodes,) bool: Dirichlet node
    node_used: np.ndarray     # (nnodes,) bool: node of a present tet
    free_edges: np.ndarray    # (n,) edge indices of free dofs, increasing
    edge_to_free: np.ndarray  # (nE,) free index or -1
    free_nodes: np.ndarray    # (m,) node ids of free nodes, increasing
    node_to_free: np.ndarray  # (nnodes,) free node index or -1

    @property
    def n(self):
        return len(self.free_edges)


def node_id(i, j, k, nx, ny):
    return i + (nx + 1) * (j + (ny + 1) * k)


def build_mesh(nx, ny, nz, h, cube_mask, dirichlet="outer") -> Mesh:
    cube_mask = np.asarray(cube_mask).astype(bool)
    assert cube_mask.size == nx * ny * nz
    cubes = np.nonzero(cube_mask)[0]
    ci = cubes % nx
    cj = (cubes // nx) % ny
    ck = cubes // (nx * ny)
    tet_ids, tet_nodes = [], []
    unit = np.eye(3, dtype=np.int64)
    for s, (a, b, _c) in enumerate(PERMS):
        p0 = np.stack([ci, cj, ck], 1)
        p1 = p0 + unit[a]
        p2 = p1 + unit[b]
        p3 = p0 + 1
        vs = [node_id(p[:, 0], p[:, 1], p[:, 2], nx, ny) for p in (p0, p1, p2, p3)]
        tet_nodes.append(np.stack(vs, 1))
        tet_ids.append(6 * cubes + s)
    tet_ids = np.concatenate(tet_ids)
    tet_nodes = np.concatenate(tet_nodes)
    order = np.argsort(tet_ids, kind="stable")
    tet_ids, tet_nodes = tet_ids[order], tet_nodes[order]
    assert np.all(np.diff(tet_nodes, axis=1) > 0)

    nnodes = (nx + 1) * (ny + 1) * (nz + 1)
    ids = np.arange(nnodes)
    ii = ids % (nx + 1)
    jj = (ids // (nx + 1)) % (ny + 1)
    kk = ids // ((nx + 1) * (ny + 1))
    node_xyz = h * np.stack([ii, jj, kk], 1).astype(np.float64)

    # edges: unique (a, b) pairs, lexicographic
    pairs = np.concatenate([tet_nodes[:, [a, b]] for a, b in LOCAL_EDGES])
    key = pairs[:, 0] * nnodes + pairs[:, 1]
    ukey, inv = np.unique(key, return_inverse=True)
    edges = np.stack([ukey // nnodes, ukey % nnodes], 1)
    T = len(tet_ids)
    tet_edges = inv.reshape(6, T).T.copy()

    # boundary faces: triangles belonging to exactly one present tet
    faces = np.concatenate([tet_nodes[:, list(f)] for f in LOCAL_FACES])
    fkey = (faces[:, 0] * nnodes + faces[:, 1]) * nnodes + faces[:, 2]
    uf, cnt = np.unique(fkey, return_counts=True)
    bfaces_key = uf[cnt == 1]
    bf = np.stack([bfaces_key // (nnodes * nnodes), (bfaces_key // nnodes) % nnodes,
                   bfaces_key % nnodes], 1)
    if dirichlet == "none":
        dfaces = bf[:0]
    elif dirichlet == "all":
        dfaces = bf
    elif dirichlet == "outer":
        grid = np.stack([ii, jj, kk], 1)
        ext = np.array([nx, ny, nz])
        g = grid[bf]                                   # (F, 3 verts, 3 coords)
        on_outer = np.zeros(len(bf), bool)
        for d in range(3):
            on_outer |= np.all(g[:, :, d] == 0, axis=1)
            on_outer |= np.all(g[:, :, d] == ext[d], axis=1)
        dfaces = bf[on_outer]
    else:
        raise ValueError(dirichlet)
    node_dir = np.zeros(nnodes, bool)
    node_dir[dfaces.ravel()] = True
    ekey_all = edges[:, 0] * nnodes + edges[:, 1]
    dkeys = np.concatenate([dfaces[:, 0] * nnodes + dfaces[:, 1],
                            dfaces[:, 0] * nnodes + dfaces[:, 2],
                            dfaces[:, 1] * nnodes + dfaces[:, 2]])
    edge_dir = np.isin(ekey_all, dkeys)

    node_used = np.zeros(nnodes, bool)
    node_used[tet_nodes.ravel()] = True
    free_edges = np.nonzero(~edge_dir)[0]
    edge_to_free = -np.ones(len(edges), np.int64)
    edge_to_free[free_edges] = np.arange(len(free_edges))
    free_nodes = np.nonzero(node_used & ~node_dir)[0]
    node_to_free = -np.ones(nnodes, np.int64)
    node_to_free[free_nodes] = np.arange(len(free_nodes))
    return Mesh(nx, ny, nz, h, node_xyz, tet_ids, tet_nodes, edges, tet_edges,
                edge_dir, node_dir, node_used, free_edges, edge_to_free,
                free_nodes, node_to_free)


def mesh_of(w) -> Mesh:
    return build_mesh(w.nx, w.ny, w.nz, w.h, w.cube_mask, w.dirichlet)
