"""Pins of the oracle's decomposition, coarse space, preconditioner and PCG
against PAPER.md's identities (PoU eq. 2.1, Lemmas 2.1/2.2, Def. 2.4
projection algebra, GEVP 3.5, Theorem 3.9 bound) and against textbook results
(dense direct solve, exact local solve in one subdomain)."""
import numpy as np
import pytest
import scipy.sparse as sp

import workloads
from oracle import assembly, coarse, dd, mesh as om, solver


@pytest.fixture(scope="module")
def c1small():
    # the c1 recipe (channels, contrast 1e4, gamma 1e-4) on an 8^3 grid, 2^3 boxes
    w = workloads.make("c1", n=8, p=2)
    return solver.Problem(w)


@pytest.fixture(scope="module")
def holes_small():
    # two through-tunnels, natural BC on their walls, mixed coefficients
    n = 8
    mask = np.ones(n ** 3, bool)
    c = np.arange(n ** 3); ci, cj, ck = c % n, (c // n) % n, c // (n * n)
    mask &= ~((cj >= 2) & (cj < 4) & (ck >= 2) & (ck < 4))      # along x
    mask &= ~((ci >= 5) & (ci < 7) & (cj >= 5) & (cj < 7))      # along z
    rng = np.random.default_rng(7)
    mu_inv = np.repeat(10 ** rng.uniform(-2, 2, n ** 3), 6)
    w = workloads.custom(n, n, n, 2, 2, 2, overlap=1, gamma=1e-3, mask=mask.astype(np.uint8),
                         mu_inv=mu_inv)
    return solver.Problem(w)


def test_partition_of_unity(c1small):
    P = c1small
    s = np.zeros(P.n)
    for d, D in zip(P.dec.dofs, P.dec.pou):
        s[d] += D
    assert np.abs(s - 1).max() <= 4 * np.finfo(float).eps
    r = np.random.default_rng(0).standard_normal(P.n)
    back = np.zeros(P.n)
    for d, D in zip(P.dec.dofs, P.dec.pou):
        back[d] += D * r[d]
    np.testing.assert_allclose(back, r, rtol=1e-15, atol=1e-15)


def test_overlap_is_two_elements_wide():
    # §4: "one layer of elements is added in each direction; this results in an
    # overlap region of two elements width between neighbouring subdomains"
    w = workloads.custom(8, 2, 2, 2, 1, 1, overlap=1)
    m = om.mesh_of(w)
    dec = dd.decompose(m, 2, 1, 1, 1)
    shared = np.intersect1d(dec.sub_tets[0], dec.sub_tets[1])
    cubes = np.unique(m.tet_ids[shared] // 6)
    assert sorted(set(cubes % 8)) == [3, 4]


def test_nonoverlapping_neumann_matrices_sum_to_A():
    # with overlap 0 the elements are partitioned, so sum_i R_i^T A_i^Neu R_i = A
    w = workloads.make("c1", n=8, p=2)
    w = workloads.with_(w, overlap=0)
    m = om.mesh_of(w)
    A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
    dec = dd.decompose(m, 2, 2, 2, 0)
    S = sp.csr_matrix(A.shape)
    for d, An in zip(dec.dofs, dd.neumann_matrices(m, w.mu_inv, w.eps, w.gamma, dec)):
        R = dd.restriction(A.shape[0], d)
        S = S + R.T @ An @ R
    assert abs(S - A).max() <= 1e-12 * abs(A).max()


def test_lemma_2_1_and_2_2(c1small):
    P = c1small
    k0 = dd.k0(P.A, P.dec)
    k1 = dd.k1(P.mesh, P.dec)
    rng = np.random.default_rng(1)
    for _ in range(10):
        U = rng.standard_normal(P.n)
        lhs = sum(U[d] @ (An @ U[d]) for d, An in zip(P.dec.dofs, P.Aneu))
        assert lhs <= k1 * (U @ (P.A @ U)) * (1 + 1e-12)
        Ui = [rng.standard_normal(len(d)) for d in P.dec.dofs]
        tot = np.zeros(P.n)
        for d, u in zip(P.dec.dofs, Ui):
            tot[d] += u
        rhs = sum(u @ (P.A[d][:, d] @ u) for d, u in zip(P.dec.dofs, Ui))
        assert tot @ (P.A @ tot) <= k0 * rhs * (1 + 1e-12)


def test_local_gradient_basis_keeps_span(holes_small):
    P = holes_small
    for d in P.dec.dofs:
        cols, Gi = coarse.local_gradient_basis(P.C, d)
        full = P.C[d].toarray()
        full = full[:, np.abs(full).sum(0) > 0]
        r = np.linalg.matrix_rank(full)
        assert Gi.shape[1] == r == np.linalg.matrix_rank(Gi.toarray())


def test_xi_projection_algebra(holes_small):
    P = holes_small
    d = P.dec.dofs[3]
    Ai = P.A[d][:, d].toarray()
    _, Gi = coarse.local_gradient_basis(P.C, d)
    G = Gi.toarray()
    xi = coarse.xi_projection(Ai, G)
    rng = np.random.default_rng(2)
    v = rng.standard_normal(len(d))
    nv = np.sqrt(v @ Ai @ v)
    assert np.sqrt(((xi @ xi @ v - xi @ v) @ Ai @ (xi @ xi @ v - xi @ v))) <= 1e-9 * nv
    np.testing.assert_allclose(xi @ G, G, atol=1e-9)
    # (I - xi) v is A_i-orthogonal to span G
    assert np.abs(G.T @ Ai @ (v - xi @ v)).max() <= 1e-9 * np.abs(G.T @ Ai @ v).max()


def test_geneo_eigenpairs(holes_small):
    P = holes_small
    i = 0
    d = P.dec.dofs[i]
    Ai = P.A[d][:, d]
    _, Gi = coarse.local_gradient_basis(P.C, d)
    lam, V, W = coarse.geneo_local(Ai, P.Aneu[i], P.dec.pou[i], Gi, 1.0)
    Ad, Bd = Ai.toarray(), P.Aneu[i].toarray()
    xi = coarse.xi_projection(Ad, Gi.toarray())
    DP = P.dec.pou[i][:, None] * (np.eye(len(d)) - xi)
    L = DP.T @ Ad @ DP
    assert np.all(lam > 1.0)
    for k in range(len(lam)):
        res = L @ V[:, k] - lam[k] * (Bd @ V[:, k])
        assert np.linalg.norm(res) <= 1e-8 * np.linalg.norm(L @ V[:, k])
    # the local near-kernel has lambda = 0: L G_i = 0
    assert np.abs(L @ Gi.toarray()).max() <= 1e-9 * np.abs(L).max()


def test_snk_rank_and_contains_nk(c1small):
    P = c1small
    cs = P.cs
    Zg = cs.Z[:, np.nonzero(cs.kinds == 0)[0]].toarray()
    assert np.linalg.matrix_rank(Zg) == cs.grad_rank
    # V_G contains the global gradients G = range C (sum_i R_i^T D_i R_i = I)
    Q, _ = np.linalg.qr(Zg @ cs.basis[:Zg.shape[1], :cs.grad_rank])
    Cd = P.C.toarray()
    assert np.abs(Cd - Q @ (Q.T @ Cd)).max() <= 1e-10
    # and is strictly larger than NK (§4: "SNK space is strictly larger")
    assert cs.grad_rank > P.C.shape[1]


def test_single_subdomain_snk_equals_nk():
    w = workloads.custom(4, 4, 4, 1, 1, 1, overlap=1, gamma=1e-2)
    P = solver.Problem(w)
    assert P.cs.grad_rank == P.C.shape[1]


def test_coarse_projection_algebra(c1small):
    P = c1small
    A = P.A
    rng = np.random.default_rng(3)
    M = P.M_inv
    u = rng.standard_normal(P.n)
    p0u = M.q(A @ u)
    p0p0u = M.q(A @ p0u)
    nA = lambda x: np.sqrt(x @ (A @ x))
    assert nA(p0p0u - p0u) <= 1e-8 * nA(u)
    Z = P.cs.Z @ P.cs.basis
    for j in rng.choice(Z.shape[1], 5, replace=False):
        z = np.asarray(Z[:, j]).ravel()
        assert nA(M.q(A @ z) - z) <= 1e-8 * nA(z)
    v = rng.standard_normal(P.n)
    assert abs((A @ M.q(A @ u)) @ v - u @ (A @ M.q(A @ v))) <= 1e-9 * nA(u) * nA(v)


@pytest.mark.parametrize("which,tol", [("c0", 1e-12), ("c1small", 1e-7)])
def test_preconditioner_symmetric(which, tol, c1small):
    # exact symmetry; in fp64 the defect is ~ cond(A_i) * eps (cond(A_i) ~ 1e3 for
    # c0, ~1e9 for the contrast-1e4 / gamma-1e-4 c1 recipe), hence the tolerances
    P = c1small if which == "c1small" else solver.Problem(workloads.make("c0"))
    rng = np.random.default_rng(4)
    for variant in ["as1", "as2", "additive"]:
        M = solver.Schwarz(P.A, P.dec, P.cs, variant=variant)
        u, v = rng.standard_normal(P.n), rng.standard_normal(P.n)
        Mu, Mv = M(u), M(v)
        assert abs(v @ Mu - u @ Mv) <= tol * np.linalg.norm(Mu) * np.linalg.norm(v)


def test_theorem_3_9_spectral_bounds(holes_small):
    # kappa(M_AS,2^{-1} A) <= (1 + k1 tau) k0 with eigenvalues in [1/(1+k1 tau), k0]
    P = holes_small
    A = P.A.toarray()
    Mi = np.stack([P.M_inv(e) for e in np.eye(P.n)], 1)
    ev = np.linalg.eigvals(Mi @ A).real
    k0, k1 = dd.k0(P.A, P.dec), dd.k1(P.mesh, P.dec)
    assert ev.min() >= 1.0 / (1.0 + k1 * P.tau) - 1e-6
    assert ev.max() <= k0 + 1e-6


def test_pcg_matches_dense_direct_solve():
    w = workloads.custom(4, 4, 4, 2, 2, 1, overlap=1, gamma=1e-2, f_seed=5)
    P = solver.Problem(w)
    f = workloads.rhs(P.n, 5)
    x, it, hist = P.solve(f, tol=1e-12)
    xd = np.linalg.solve(P.A.toarray(), f)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)
    assert hist[-1] <= 1e-12


def test_pcg_single_subdomain_is_exact():
    # N = 1: M_AS = A^{-1}, so CG converges in one iteration
    w = workloads.custom(3, 3, 3, 1, 1, 1, overlap=1, gamma=1e-2)
    P = solver.Problem(w)
    f = workloads.rhs(P.n, 1)
    x, it, _ = P.solve(f, tol=1e-10)
    assert it == 1


def test_pcg_zero_rhs():
    w = workloads.custom(3, 3, 3, 1, 1, 1)
    P = solver.Problem(w, coarse_on=False)
    x, it, _ = P.solve(np.zeros(P.n))
    assert it == 0 and not x.any()


def test_c0_geneo_empty_like_table1():
    # PAPER.md Table 1 ("GenEO size 0") for the homogeneous Dirichlet problem at
    # tau = 10; here configs[0] (homogeneous cube, Dirichlet, threshold 0.1 = 1/tau)
    w = workloads.make("c0")
    P = solver.Problem(w)
    assert sum(len(l) for l in P.cs.geneo_lambdas) == 0
    f = workloads.rhs(P.n, w.f_seed)
    _, it2, _ = P.solve(f)
    _, it1, _ = solver.pcg(P.A, f, solver.Schwarz(P.A, P.dec, None, "as1"))
    assert it2 < it1


def test_coarse_start_balancing_identity():
    """Reading R13, the algebra.  For a Z-orthogonal residual (Z^T r = 0, which
    PCG keeps for every k from x0 = Q f) Q r = 0, and eq. (2.4) equals both
    (I - Q A) M_AS r and the one-coarse-solve form M_AS r + Q (r - A M_AS r).
    On c0 (E well conditioned) the three agree to rounding; on a generic r they
    do not (the identity needs the start)."""
    P = solver.Problem(workloads.make("c0"))
    M = P.M_inv
    rng = np.random.default_rng(12)
    v = rng.standard_normal(P.n)
    r = v - P.A @ M.q(v)                           # Z^T r = 0
    Z = P.cs.Z @ P.cs.basis
    assert np.linalg.norm(Z.T @ r) <= 1e-10 * np.linalg.norm(Z.T @ v)
    full = M(r)
    w = M.m_as(r)
    one_solve = w + M.q(r - P.A @ w)
    reduced = w - M.q(P.A @ w)
    assert np.linalg.norm(one_solve - full) <= 1e-11 * np.linalg.norm(full)
    # without the +Q r term the rounding left in Z^T r (~1e-12) is not corrected
    # but amplified by the local solves: agreement only to ~1e-8 even on c0
    assert np.linalg.norm(reduced - full) <= 1e-6 * np.linalg.norm(full)
    wv = M.m_as(v)
    assert np.linalg.norm(wv + M.q(v - P.A @ wv) - M(v)) > 1e-7 * np.linalg.norm(M(v))


def test_coarse_start_trajectory(c1small):
    """Reading R13 on the contrast-1e4 / gamma-1e-4 recipe (kappa(E) ~ 1e11):
    PCG with eq. (2.4) from x0 = Q f, from x0 = 0, and with the one-coarse-solve
    form M_AS r + Q (r - A M_AS r) from x0 = Q f take the same number of
    iterations and reach the same solution (the form without the +Q r term
    would stall here: rounding leaves Z^T r_k ~ 1e-8, amplified by E^{-1})."""
    P = c1small
    M = P.M_inv
    f = workloads.rhs(P.n, 11)
    xz, itz, _ = P.solve(f)
    xc, itc, hc = P.solve(f, x0="coarse")

    def one_solve(r):
        w = M.m_as(r)
        return w + M.q(r - P.A @ w)

    xa, ita, ha = solver.pcg(P.A, f, one_solve, x0=M.q(f))
    assert hc[-1] <= 1e-8 and ha[-1] <= 1e-8
    assert abs(itc - itz) <= 1 and abs(ita - itc) <= 1
    assert np.linalg.norm(xa - xc) <= 1e-8 * np.linalg.norm(xc)
    # different starts: both residuals <= 1e-8, forward errors differ (~1e-6 here)
    assert np.linalg.norm(xc - xz) <= 1e-5 * np.linalg.norm(xz)


def test_pcg_coarse_start_matches_dense_direct_solve():
    w = workloads.custom(4, 4, 4, 2, 2, 1, overlap=1, gamma=1e-2, f_seed=5)
    P = solver.Problem(w)
    f = workloads.rhs(P.n, 5)
    x, it, hist = P.solve(f, tol=1e-12, x0="coarse")
    xd = np.linalg.solve(P.A.toarray(), f)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)
    assert hist[-1] <= 1e-12


def test_geneo_pencil_deflation_keeps_the_kept_eigenpairs():
    """Reading R15 (the device solves GEVP 3.5 on {v : G_j^T B v = 0}): null(L)
    contains range(G_j) (P G_j = 0), so the eigenpairs with lambda > tau are
    B-orthogonal to range(G_j) and the deflated pencil (Q2^T L Q2, Q2^T B Q2), Q2 the
    last n - g columns of the QR factor of B G_j, has the same ones -- while its B
    is far better conditioned."""
    import scipy.linalg as sla
    import workloads
    from oracle import assembly, coarse, dd, mesh as om
    w = workloads.make("c1", n=8, p=2)
    m = om.mesh_of(w)
    A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
    C = assembly.gradient_matrix(m)
    dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
    Aneu = dd.neumann_matrices(m, w.mu_inv, w.eps, w.gamma, dec)
    tau = 1.0 / w.threshold
    for i in (0, 3):
        d = dec.dofs[i]
        cols, Gi = coarse.local_gradient_basis(C, d)
        lam, V, _ = coarse.geneo_local(A[d][:, d].tocsr(), Aneu[i], dec.pou[i], Gi, tau)
        Ad, B, G = A[d][:, d].toarray(), Aneu[i].toarray(), Gi.toarray()
        P = np.eye(len(d)) - coarse.xi_projection(Ad, G)
        DP = dec.pou[i][:, None] * P
        L = DP.T @ Ad @ DP
        L = 0.5 * (L + L.T)
        assert np.abs(L @ G).max() <= 1e-9 * np.abs(L).max()          # range(G) in null(L)
        assert np.abs(G.T @ B @ V).max() <= 1e-8 * np.abs(B @ V).max()  # kept V B-orthogonal to it
        Q, _ = sla.qr(B @ G, mode="full")
        Q2 = Q[:, G.shape[1]:]
        Lc, Bc = Q2.T @ L @ Q2, Q2.T @ B @ Q2
        lc = sla.eigh(0.5 * (Lc + Lc.T), 0.5 * (Bc + Bc.T), eigvals_only=True, subset_by_value=(tau, np.inf))
        assert len(lc) == len(lam) and np.allclose(lc, lam, rtol=1e-8, atol=0)
        assert np.linalg.cond(Bc) < 1e-3 * np.linalg.cond(B)
