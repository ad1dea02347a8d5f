"""GPU checks of setup-phase machinery that the parity cases do not isolate."""
import os

import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_row_chunked_spgemm_gives_the_same_coarse_matrix():
    """E = Z^T (A Z) and the gradient Gram are formed by row-chunked cuSPARSE
    products (bounded workspace, needed at c2 size).  Forcing tiny chunks must give
    the same E up to the summation order inside cuSPARSE (entries within 1e-14
    of the largest) and the same solve."""
    from paper_2311_18783_b200 import MaxwellDD
    w = workloads.make("c1", n=8, p=2)
    G0 = MaxwellDD(w)
    os.environ["MDD_SPGEMM_MAX_PROD"] = "20000"
    try:
        G1 = MaxwellDD(w)
    finally:
        os.environ.pop("MDD_SPGEMM_MAX_PROD", None)
    E0, E1 = G0.coarse_matrix(), G1.coarse_matrix()
    assert np.array_equal(E0.indptr, E1.indptr) and np.array_equal(E0.indices, E1.indices)
    assert np.abs(E0.data - E1.data).max() <= 1e-14 * np.abs(E0.data).max()
    f = workloads.rhs(G0.n, w.f_seed)
    x0, it0, _ = G0.solve_host(f)
    x1, it1, _ = G1.solve_host(f)
    assert it0 == it1 and np.linalg.norm(x0 - x1) <= 1e-8 * np.linalg.norm(x0)
