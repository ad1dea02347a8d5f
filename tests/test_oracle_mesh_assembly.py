"""Pins of the oracle's mesh, numbering and Whitney assembly against what the
mathematics fixes (closed-form counts, Euler characteristic, exact integrals of
fields the Whitney space reproduces, de Rham exactness, Betti numbers)."""
import itertools

import numpy as np
import pytest
import scipy.linalg as sla

import workloads
from oracle import assembly, mesh as om
from oracle.mesh import LOCAL_EDGES


def kuhn_edge_count(nx, ny, nz):
    # 3 axis families + 3 face-diagonal families + 1 body diagonal family,
    # counted on the lattice (each family's edges are translates of one vector)
    return (nx * (ny + 1) * (nz + 1) + (nx + 1) * ny * (nz + 1) + (nx + 1) * (ny + 1) * nz
            + nx * ny * (nz + 1) + nx * (ny + 1) * nz + (nx + 1) * ny * nz + nx * ny * nz)


def boundary_edge_count(nx, ny, nz):
    # each outer face is a grid of squares with one diagonal each; the 12 box
    # edges are shared by two faces
    def face(a, b):
        return a * (b + 1) + (a + 1) * b + a * b
    return 2 * (face(nx, ny) + face(nx, nz) + face(ny, nz)) - 4 * (nx + ny + nz)


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 1, 1), (2, 3, 4), (5, 5, 5), (8, 8, 8)])
def test_edge_counts_closed_form(dims):
    nx, ny, nz = dims
    m = om.build_mesh(nx, ny, nz, 1.0, np.ones(nx * ny * nz, np.uint8), "outer")
    assert len(m.edges) == kuhn_edge_count(nx, ny, nz)
    assert m.edge_dir.sum() == boundary_edge_count(nx, ny, nz)
    assert m.n == kuhn_edge_count(nx, ny, nz) - boundary_edge_count(nx, ny, nz)
    assert len(m.tet_ids) == 6 * nx * ny * nz
    # free nodes = interior lattice nodes
    assert len(m.free_nodes) == max(nx - 1, 0) * max(ny - 1, 0) * max(nz - 1, 0)


def test_c0_size_matches_baseline():
    # BASELINE configs[0]: "lowest-order Nédélec edge DOFs (~4.3k)"
    w = workloads.make("c0")
    m = om.mesh_of(w)
    assert len(m.edges) == 4184
    assert m.n == 4184 - 1152


def test_edges_oriented_and_lexicographic():
    m = om.build_mesh(3, 2, 2, 0.5, np.ones(12, np.uint8))
    assert np.all(m.edges[:, 0] < m.edges[:, 1])
    key = m.edges[:, 0] * 10 ** 6 + m.edges[:, 1]
    assert np.all(np.diff(key) > 0)
    # every tet edge maps back to its endpoints
    for t in range(len(m.tet_ids)):
        for le, (a, b) in enumerate(LOCAL_EDGES):
            e = m.tet_edges[t, le]
            assert tuple(m.edges[e]) == (m.tet_nodes[t, a], m.tet_nodes[t, b])


def _tunnel_mask(n, tunnels):
    mask = np.ones(n ** 3, bool)
    c = np.arange(n ** 3)
    ci, cj, ck = c % n, (c // n) % n, c // (n * n)
    co = (ci, cj, ck)
    for axis, la, lb, s in tunnels:
        a, b = [d for d in range(3) if d != axis]
        mask &= ~((co[a] >= la) & (co[a] < la + s) & (co[b] >= lb) & (co[b] < lb + s))
    return mask.astype(np.uint8)


def _euler(m):
    faces = set()
    for t in m.tet_nodes:
        for f in itertools.combinations(sorted(t), 3):
            faces.add(f)
    V = m.node_used.sum()
    return V - len(m.edges) + len(faces) - len(m.tet_ids)


@pytest.mark.parametrize("tunnels,chi", [([], 1), ([(0, 1, 1, 1)], 0),
                                         ([(0, 1, 1, 1), (1, 1, 3, 1)], -1)])
def test_euler_characteristic(tunnels, chi):
    # V - E + F - T = b0 - b1 + b2 for the meshed solid
    n = 5
    m = om.build_mesh(n, n, n, 1.0 / n, _tunnel_mask(n, tunnels))
    assert _euler(m) == chi


def _random_tets(rng, k):
    xyz = rng.standard_normal((k, 4, 3))
    J = np.stack([xyz[:, i] - xyz[:, 0] for i in (1, 2, 3)], 2)
    det = np.linalg.det(J)
    xyz[det < 0, 1], xyz[det < 0, 2] = xyz[det < 0, 2].copy(), xyz[det < 0, 1].copy()
    return xyz


def test_whitney_mass_reproduces_constant_fields():
    # Whitney interpolation is exact for constant fields: dof_e = c . (x_b - x_a),
    # so u^T M u' = eps |T| c . c'  (exact integral)
    rng = np.random.default_rng(0)
    xyz = _random_tets(rng, 20)
    eps = rng.uniform(0.5, 2, 20)
    Ke, Me = assembly.element_matrices(xyz, np.ones(20), eps)
    vol = np.abs(np.linalg.det(np.stack([xyz[:, i] - xyz[:, 0] for i in (1, 2, 3)], 2))) / 6
    for _ in range(5):
        c1, c2 = rng.standard_normal(3), rng.standard_normal(3)
        u1 = np.stack([(xyz[:, b] - xyz[:, a]) @ c1 for a, b in LOCAL_EDGES], 1)
        u2 = np.stack([(xyz[:, b] - xyz[:, a]) @ c2 for a, b in LOCAL_EDGES], 1)
        got = np.einsum("tm,tmn,tn->t", u1, Me, u2)
        np.testing.assert_allclose(got, eps * vol * (c1 @ c2), rtol=1e-11)
        # constant fields are gradients of linear functions: no curl energy
        assert np.abs(np.einsum("tm,tmn,tn->t", u1, Ke, u1)).max() < 1e-10 * np.abs(Ke).max()


def test_whitney_curl_energy_of_rotational_field():
    # u = 1/2 c x x has curl c; the Whitney interpolant has the same (constant)
    # curl (commuting diagram), so u^T K u = mu^{-1} |T| |c|^2 exactly.
    rng = np.random.default_rng(1)
    xyz = _random_tets(rng, 20)
    mu_inv = rng.uniform(0.1, 10, 20)
    Ke, _ = assembly.element_matrices(xyz, mu_inv, np.ones(20))
    vol = np.abs(np.linalg.det(np.stack([xyz[:, i] - xyz[:, 0] for i in (1, 2, 3)], 2))) / 6
    c = rng.standard_normal(3)
    # dof = line integral of a linear field = midpoint value . tangent
    u = np.stack([0.5 * np.cross(c, 0.5 * (xyz[:, a] + xyz[:, b])) @ np.eye(3) * 1.0
                  for a, b in LOCAL_EDGES], 1)
    u = np.einsum("tmi,tmi->tm", u,
                  np.stack([xyz[:, b] - xyz[:, a] for a, b in LOCAL_EDGES], 1))
    got = np.einsum("tm,tmn,tn->t", u, Ke, u)
    np.testing.assert_allclose(got, mu_inv * vol * (c @ c), rtol=1e-11)


def test_element_matrix_ranks():
    rng = np.random.default_rng(2)
    xyz = _random_tets(rng, 5)
    Ke, Me = assembly.element_matrices(xyz, np.ones(5), np.ones(5))
    for k in range(5):
        assert np.linalg.matrix_rank(Ke[k], tol=1e-9 * np.abs(Ke[k]).max()) == 3  # 6 - (4 - 1)
        assert np.linalg.eigvalsh(Me[k]).min() > 0


def _cases():
    n = 5
    return [
        ("box-outer", om.build_mesh(n, n, n, 1 / n, np.ones(n ** 3, np.uint8), "outer")),
        ("tunnel-outer", om.build_mesh(n, n, n, 1 / n, _tunnel_mask(n, [(0, 1, 1, 2)]), "outer")),
        ("tunnels-none", om.build_mesh(n, n, n, 1 / n, _tunnel_mask(n, [(0, 1, 1, 1), (2, 3, 1, 1)]), "none")),
        ("tunnel-all", om.build_mesh(n, n, n, 1 / n, _tunnel_mask(n, [(1, 2, 2, 1)]), "all")),
    ]


@pytest.mark.parametrize("name,m", _cases())
def test_discrete_exactness_KC_zero(name, m):
    rng = np.random.default_rng(3)
    T = 6 * m.nx * m.ny * m.nz
    mu_inv = 10 ** rng.uniform(-2, 4, T)
    K, M = assembly.assemble(m, mu_inv, np.ones(T))
    C = assembly.gradient_matrix(m)
    assert abs(K @ C).max() <= 1e-12 * abs(K).max()
    A = (K + 1e-3 * M).toarray()
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    assert np.linalg.eigvalsh(A).min() > 0


@pytest.mark.parametrize("tunnels,mode,harmonic", [
    ([], "none", 0), ([(0, 1, 1, 1)], "none", 1), ([(0, 1, 1, 1), (1, 1, 3, 1)], "none", 2),
    ([(0, 1, 1, 1), (1, 1, 3, 1)], "outer", 0), ([(0, 1, 1, 1)], "all", 0),
])
def test_harmonic_fields_equal_betti(tunnels, mode, harmonic):
    # dim ker K - rank C = dim of discrete harmonic fields: b1 (holes) with natural
    # BC, the relative b1(Omega, Gamma_D) = 0 for tunnels ending on a Dirichlet box.
    n = 5
    m = om.build_mesh(n, n, n, 1 / n, _tunnel_mask(n, tunnels), mode)
    K, _ = assembly.assemble(m, np.ones(6 * n ** 3), np.ones(6 * n ** 3))
    C = assembly.gradient_matrix(m)
    w = np.linalg.eigvalsh(K.toarray())
    dimker = int((w < 1e-9 * w.max()).sum())
    rankC = np.linalg.matrix_rank(C.toarray())
    assert dimker - rankC == harmonic


def test_cavity_gives_dirichlet_harmonic_field():
    # b2 = 1 (an enclosed void) -> one harmonic field under E x n = 0 everywhere
    n = 5
    mask = np.ones(n ** 3, np.uint8)
    mask[2 + n * (2 + n * 2)] = 0
    m = om.build_mesh(n, n, n, 1 / n, mask, "all")
    K, _ = assembly.assemble(m, np.ones(6 * n ** 3), np.ones(6 * n ** 3))
    C = assembly.gradient_matrix(m)
    w = np.linalg.eigvalsh(K.toarray())
    assert int((w < 1e-9 * w.max()).sum()) - np.linalg.matrix_rank(C.toarray()) == 1


def test_global_energies_of_exact_fields_pin_coefficient_map():
    # with natural BC every edge is a dof: the constant field has energy
    # sum_T eps_T |T| |c|^2 and the rotational field sum_T mu_T^{-1} |T| |c|^2,
    # |T| = h^3 / 6 for every Kuhn tet.  Pins per-tet coefficient indexing.
    n, h = 3, 0.25
    rng = np.random.default_rng(4)
    mask = np.ones(n ** 3, np.uint8); mask[4] = 0
    m = om.build_mesh(n, n, n, h, mask, "none")
    T = 6 * n ** 3
    mu_inv, eps = rng.uniform(0.5, 2, T), rng.uniform(0.5, 2, T)
    K, M = assembly.assemble(m, mu_inv, eps)
    c = rng.standard_normal(3)
    x = m.node_xyz
    e = m.edges[m.free_edges]
    u_const = (x[e[:, 1]] - x[e[:, 0]]) @ c
    mid = 0.5 * (x[e[:, 0]] + x[e[:, 1]])
    u_rot = np.einsum("ki,ki->k", 0.5 * np.cross(c, mid), x[e[:, 1]] - x[e[:, 0]])
    present = m.tet_ids
    np.testing.assert_allclose(u_const @ (M @ u_const), eps[present].sum() * h ** 3 / 6 * (c @ c), rtol=1e-12)
    np.testing.assert_allclose(u_rot @ (K @ u_rot), mu_inv[present].sum() * h ** 3 / 6 * (c @ c), rtol=1e-12)
