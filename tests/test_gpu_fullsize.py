"""GPU checks at BASELINE's full c1 size, where the oracle cannot run end to end
(its SNK basis needs a dense eigendecomposition of the 64k-column candidate
Gram): kappa-free backward errors of every subdomain solve, of the coarse solve
and of the PCG solution against the oracle's own A; forward errors of sampled
subdomain solves against the extended-precision reference; properties that hold
at any size (P0 = QA is an A-orthogonal projection, M symmetric).  The oracle's
own answers at the bench's 4^3 partition come from the 16^3 goldens
(tests/test_gpu_golden.py)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads
from oracle import assembly, dd, mesh as om

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    from paper_2311_18783_b200 import MaxwellDD
    w = workloads.make("c1")
    G = MaxwellDD(w)
    m = om.mesh_of(w)
    A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
    dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
    return w, G, A.tocsr(), dec


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def test_assembled_matrix_full_size(c1):
    w, G, A, dec = c1
    assert np.array_equal(G.int_array("A_ptr"), A.indptr)
    assert np.abs(G.double_array("A_val") - A.data).max() <= 1e-13 * np.abs(A.data).max()


def test_every_local_solve_is_backward_stable_full_size(c1):
    """All 64 subdomain solves A_i x_i = R_i r of the full-size c1 (the bench's
    configuration), through mdd_apply_local_parts: normwise backward error at most
    8 eps on every subdomain (kappa-free: kappa(A_i) ~ 1e11 here), and on three
    subdomains the forward error against the extended-precision reference is at
    most 4x that of the oracle's own fp64 direct solver (SuperLU)."""
    from oracle import refine
    from parity_lib import EPS, backward_error, rel_ld
    w, G, A, dec = c1
    r = np.random.default_rng(11).standard_normal(A.shape[0])
    xl = torch.empty(int(G.info["nloc"]), dtype=torch.float64, device="cuda")
    G.apply_local_parts(dev(r), xl)
    xl = xl.cpu().numpy()
    sp_ = G.int_array("sub_ptr")
    worst = 0.0
    for i, d in enumerate(dec.dofs):
        assert np.array_equal(G.int_array("sub_dofs")[sp_[i]:sp_[i + 1]], d)
        Ai = A[d][:, d].tocsr()
        worst = max(worst, backward_error(Ai, xl[sp_[i]:sp_[i + 1]], r[d]))
    assert worst <= 8 * EPS, worst
    for i in (0, 21, 63):
        d = dec.dofs[i]
        Ai = A[d][:, d].tocsr()
        lu = spla.splu(Ai.tocsc())
        xr = refine.refined_solve(Ai, r[d], lu)
        e_gpu = rel_ld(xl[sp_[i]:sp_[i + 1]], xr)
        e_lu = rel_ld(lu.solve(r[d]), xr)
        assert e_gpu <= 4 * max(e_lu, EPS), (i, e_gpu, e_lu)


def test_coarse_solve_backward_error_full_size(c1):
    """E y = v on the full-size c1 coarse matrix (n0 ~ 51k, kappa ~ 1e13): the
    normwise backward error of the device's static-pivot supernodal LDL^T with
    partitioned-inverse panels, at 10x the observation on the same machine
    (it is larger than a dense Cholesky's, ~1e-12 vs 1e-17)."""
    from parity_lib import backward_error
    w, G, A, dec = c1
    n0 = int(G.info["n0"])
    E = G.coarse_matrix()
    v = np.random.default_rng(12).standard_normal(n0)
    y = torch.empty(n0, dtype=torch.float64, device="cuda")
    G.apply_coarse_inverse(dev(v), y)
    be = backward_error(E, y.cpu().numpy(), v)
    print(f"c1 full-size coarse backward error {be:.2e}")
    assert be <= 1e-11, be


def test_coarse_projection_properties(c1):
    w, G, A, dec = c1
    n = A.shape[0]
    rng = np.random.default_rng(5)
    v = rng.standard_normal(n)

    def Q(x):
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        G.apply_coarse(dev(x), y)
        return y.cpu().numpy()

    p = Q(A @ v)
    pp = Q(A @ p)
    nA = lambda x: np.sqrt(x @ (A @ x))
    assert nA(pp - p) <= 1e-5 * nA(p)          # P0^2 = P0 (kappa(E) ~ 1e13, static pivots)
    u = rng.standard_normal(n)
    assert abs(u @ Q(v) - v @ Q(u)) <= 1e-10 * np.linalg.norm(Q(v)) * np.linalg.norm(u)


def test_pcg_full_size(c1):
    """Full-size c1 PCG: converged, bit-reproducible, and the solution's normwise
    backward error ||f - A x|| / (||A|| ||x|| + ||f||) (kappa-free) is below
    1e-12: the iterate solves a nearby system, whatever kappa(A) ~ 1e11 does to
    its forward error; the true relative residual is reported beside it."""
    from parity_lib import backward_error
    w, G, A, dec = c1
    f = workloads.rhs(A.shape[0], w.f_seed)
    x = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
    it, rel, ok = G.solve(dev(f), x, tol=1e-8)
    assert ok and rel <= 1e-8 and 10 <= it <= 200
    xh = x.cpu().numpy()
    be = backward_error(A, xh, f)
    tr = np.linalg.norm(f - A @ xh) / np.linalg.norm(f)
    print(f"c1 full size: {it} iterations, backward error {be:.2e}, true relative residual {tr:.2e}")
    assert be <= 1e-12, be
    it2, rel2, ok2 = G.solve(dev(f), x, tol=1e-8)
    assert it2 == it and np.array_equal(x.cpu().numpy(), xh)   # bit-reproducible


def test_pcg_full_size_coarse_start(c1):
    """Reading R13 at full size: the one-coarse-solve loop from x0 = Q f takes the
    iteration count of eq. (2.4) from x0 = 0 (+-1), reaches the same true
    residual level and is bit-reproducible."""
    w, G, A, dec = c1
    f = workloads.rhs(A.shape[0], w.f_seed)
    x = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
    it0, _, _ = G.solve(dev(f), x, tol=1e-8)
    x0 = x.cpu().numpy()
    G.set_variant("as2_coarse_start")
    try:
        it, rel, ok = G.solve(dev(f), x, tol=1e-8)
        xh = x.cpu().numpy()
        it2, _, _ = G.solve(dev(f), x, tol=1e-8)
        assert it2 == it and np.array_equal(x.cpu().numpy(), xh)
    finally:
        G.set_variant("as2")
    assert ok and rel <= 1e-8 and abs(it - it0) <= 1
    from parity_lib import backward_error
    assert backward_error(A, xh, f) <= 1e-12
    # the two loops' solutions differ by the fp64 solvers' own accuracy at kappa ~ 1e11
    # (the golden runs at 16^3 show 5e-6 between device and oracle)
    assert np.linalg.norm(xh - x0) <= 1e-4 * np.linalg.norm(x0)


def test_sweep_is_grid_independent_and_reproducible():
    # the persistent sweep's partial sums are combined in a fixed order, so the
    # result must not depend on how many CTAs run it (a race or a shared-memory
    # overrun shows up here first); MDD_SWEEP_GRID caps the persistent grid
    import os
    from paper_2311_18783_b200 import MaxwellDD
    w = workloads.make("c1", n=16, p=4)
    outs = {}
    for grid in ("0", "5"):
        os.environ["MDD_SWEEP_GRID"] = grid
        try:
            G = MaxwellDD(w)
        finally:
            os.environ.pop("MDD_SWEEP_GRID", None)
        g = torch.Generator(device="cuda").manual_seed(0)
        v = torch.randn(G.n, dtype=torch.float64, device="cuda", generator=g)
        y = [torch.empty_like(v) for _ in range(3)]
        G.apply_local(v, y[0])
        G.apply_coarse(v, y[1])
        G.apply_preconditioner(v, y[2])
        outs[grid] = [t.cpu().numpy() for t in y]
        # repeated applications (the few-CTA grid streams many tasks per CTA
        # through the descriptor / tile rings: the race-prone regime)
        for _ in range(10):
            G.apply_preconditioner(v, y[0])
            assert np.array_equal(y[0].cpu().numpy(), outs[grid][2])
        G.close()
    for name, a, b in zip(("local", "coarse", "preconditioner"), outs["0"], outs["5"]):
        assert np.array_equal(a, b), f"{name}: max rel diff {np.abs(a - b).max() / np.abs(a).max():.3e}"


def _geneo_golden(cfg):
    import json
    import os
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"geneo_{cfg}_full.json")
    return json.load(open(p)) if os.path.exists(p) else None


def test_geneo_counts_full_size_c1(c1):
    """GenEO counts of every subdomain of the full-size c1 bit-exact against the
    oracle's per-subdomain dense GEVPs (tests/golden/geneo_c1_full.json).  The kept
    eigenvalues: GEVP 3.5 (eq. 3.1) at contrast 1e4, gamma = 1e-4 moves
    them by up to 2.2e-4 relative when the ORACLE itself only sums the element
    matrices in another order (tests/golden/geneo_c1_full_order_sensitivity.json,
    tools/geneo_order_sensitivity.py; the device's slot-ordered assembly is one more
    such order).  Tolerance: 10x that measured sensitivity on the subdomains the
    channels cross.  On the subdomains whose oracle eigenvalues did not move
    (< 1e-12) the device's own algorithm sets the scale: it solves the pencil on
    the B-orthogonal complement of range(G_j) (reading R15) through a basis with
    kappa ~ 6e6, so its eigenvalues carry eps * kappa ~ 1e-9 relative to the
    largest one -- per eigenvalue 1e-9 (1 + lambda_max / lambda) (subdomain 7:
    4.2e-8 observed on lambda_max / lambda_min = 110)."""
    import json
    import os
    g = _geneo_golden("c1")
    if g is None or len(g["count"]) < g["nsub"]:
        pytest.skip("geneo_c1_full golden not generated")
    sens = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                       "geneo_c1_full_order_sensitivity.json")))["max_rel"]
    w, G, A, dec = c1
    cnt = [int(c) for c in G.int_array("geneo_count")]
    assert cnt == [g["count"][str(i)] for i in range(g["nsub"])]
    lam = G.double_array("geneo_lambda")
    smax = max(sens.values())
    off = 0
    for i in range(g["nsub"]):
        lo = np.asarray(g["lambda"][str(i)])
        li = lam[off:off + cnt[i]]
        off += cnt[i]
        if not len(lo):
            continue
        r = np.abs(li - lo) / lo
        if sens[str(i)] < 1e-12:
            k = int(np.argmax(r / (1 + lo.max() / lo)))
            assert r[k] <= 1e-9 * (1 + lo.max() / lo[k]), (i, r[k], lo[k], lo.max())
        else:
            assert r.max() <= 10 * smax, (i, r.max(), sens[str(i)])


@pytest.fixture(scope="module")
def c2():
    from paper_2311_18783_b200 import MaxwellDD
    w = workloads.make("c2")
    G = MaxwellDD(w, variant="as2_coarse_start")
    m = om.mesh_of(w)
    A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
    dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
    return w, G, A.tocsr(), dec


def test_c2_full_size(c2):
    """BASELINE config 3 (c2) at full size: 48^3 cubes minus two 8x8 through-holes
    (Betti 2, natural BC on the hole walls), 216 subdomains, gamma = 1e-6, mu / eps
    per subdomain over four decades.  GenEO counts of every subdomain bit-exact
    against the oracle's per-subdomain GEVPs (tests/golden/geneo_c2_full.json),
    every local solve backward stable, and the PCG of the bench's loop converging
    with a backward-stable solution (the coarse matrix drops its numerically
    dependent directions, reading R11)."""
    from parity_lib import EPS, backward_error
    w, G, A, dec = c2
    g = _geneo_golden("c2")
    if g is not None and len(g["count"]) == g["nsub"]:
        assert [int(c) for c in G.int_array("geneo_count")] == [g["count"][str(i)] for i in range(g["nsub"])]
    r = np.random.default_rng(21).standard_normal(A.shape[0])
    xl = torch.empty(int(G.info["nloc"]), dtype=torch.float64, device="cuda")
    G.apply_local_parts(dev(r), xl)
    xl = xl.cpu().numpy()
    sp_ = G.int_array("sub_ptr")
    worst = max(backward_error(A[d][:, d].tocsr(), xl[sp_[i]:sp_[i + 1]], r[d]) for i, d in enumerate(dec.dofs))
    assert worst <= 8 * EPS, worst
    f = workloads.rhs(A.shape[0], w.f_seed)
    x = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
    it, rel, ok = G.solve(dev(f), x, tol=1e-8)
    xh = x.cpu().numpy()
    be = backward_error(A, xh, f)
    print(f"c2 full size: {it} iterations, dropped coarse pivots {G.info['coarse_perturbed']}, "
          f"solution backward error {be:.2e}")
    assert ok and rel <= 1e-8 and np.isfinite(xh).all() and be <= 1e-12


def test_c3_one_gpu_share():
    """BASELINE config 4 (c3) at ONE GPU's share of its 8-GPU mesh: 48^3 cubes
    (an eighth of 96^3) with 4^3 subdomains of the full config's size (12^3 cubes
    each + 2 overlap layers -> ~30k local dofs, the block-Lanczos GenEO path),
    16 z-layers of mu^-1 in {1, 1e3}, per-element eps, gamma = 1e-3.  The full 96^3
    mesh needs the distributed setup (DESIGN.md §9/§10).  Every local solve backward
    stable, PCG of the bench's loop to 1e-8 with a backward-stable solution.  The
    oracle cannot run this size; the iteration count (41 observed on the B200,
    n = 753,552, n0 = 149,733, 3,681 GenEO vectors; the 12^3 recipe takes 28 on both
    sides; Tables 3-7 report 23-28 for AS-SNK-GenEO on its beams) is held
    to a loose bound of 60 only to catch a broken coarse space."""
    from paper_2311_18783_b200 import MaxwellDD
    from parity_lib import EPS, backward_error
    w = workloads.make("c3", n=48, p=4)
    G = MaxwellDD(w, variant="as2_coarse_start")
    m = om.mesh_of(w)
    A = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)[0].tocsr()
    dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
    assert G.n == A.shape[0] and w.overlap == 2
    r = np.random.default_rng(31).standard_normal(G.n)
    xl = torch.empty(int(G.info["nloc"]), dtype=torch.float64, device="cuda")
    G.apply_local_parts(dev(r), xl)
    xl = xl.cpu().numpy()
    sp_ = G.int_array("sub_ptr")
    assert np.array_equal(np.diff(sp_), [len(d) for d in dec.dofs])
    worst = max(backward_error(A[d][:, d].tocsr(), xl[sp_[i]:sp_[i + 1]], r[d])
                for i, d in list(enumerate(dec.dofs))[::7])
    assert worst <= 8 * EPS, worst
    f = workloads.rhs(G.n, w.f_seed)
    x = torch.empty(G.n, dtype=torch.float64, device="cuda")
    it, rel, ok = G.solve(dev(f), x, tol=1e-8)
    xh = x.cpu().numpy()
    be = backward_error(A, xh, f)
    print(f"c3 one-GPU share: n={G.n} n0={G.info['n0']} geneo={G.info['ngeneo']} {it} iterations, "
          f"dropped coarse pivots {G.info['coarse_perturbed']}, solution backward error {be:.2e}")
    assert ok and rel <= 1e-8 and it <= 60 and be <= 1e-12
    G.close()
