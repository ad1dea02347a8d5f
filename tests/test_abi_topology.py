"""CPU tests of the C-ABI library: it loads, exports every symbol the header
declares, and its host-side integer work (numbering, pattern of A, subdomain
dof lists N_i, G_i columns) is bit-identical to the oracle's."""
import re
import os

import numpy as np
import pytest

import workloads
from oracle import assembly, coarse, dd, mesh as om

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2311_18783_b200 import _lib
    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "maxwell_dd.h")).read()
    declared = set(re.findall(r"\b(mdd_[a-z_]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def _cases():
    n = 6
    mask = np.ones(n ** 3, bool)
    c = np.arange(n ** 3); ci, cj, ck = c % n, (c // n) % n, c // (n * n)
    mask &= ~((cj >= 2) & (cj < 4) & (ck >= 1) & (ck < 3))
    return [
        ("c0", workloads.make("c0")),
        ("c1-recipe-8", workloads.make("c1", n=8, p=2)),
        ("holes-outer", workloads.custom(n, n, n, 2, 3, 1, overlap=1, mask=mask.astype(np.uint8))),
        ("holes-all-ov2", workloads.custom(n, n, n, 3, 1, 2, overlap=2, mask=mask.astype(np.uint8),
                                            dirichlet="all")),
        ("box-none", workloads.custom(4, 3, 2, 2, 1, 1, overlap=1, dirichlet="none")),
        ("ragged-1sub", workloads.custom(5, 3, 7, 1, 1, 1, overlap=1)),
    ]


@pytest.mark.parametrize("name,w", _cases())
def test_topology_bit_exact(name, w):
    from paper_2311_18783_b200 import topology_array as T
    m = om.mesh_of(w)
    assert np.array_equal(T(w, "edge_tail"), m.edges[:, 0])
    assert np.array_equal(T(w, "edge_head"), m.edges[:, 1])
    assert np.array_equal(T(w, "free_edges"), m.free_edges)
    assert np.array_equal(T(w, "free_nodes"), m.free_nodes)
    A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
    assert np.array_equal(T(w, "A_ptr"), A.indptr)
    assert np.array_equal(T(w, "A_idx"), A.indices)
    dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
    ptr = T(w, "sub_ptr")
    dofs = T(w, "sub_dofs")
    assert len(ptr) == dec.nsub + 1
    for i, d in enumerate(dec.dofs):
        assert np.array_equal(dofs[ptr[i]:ptr[i + 1]], d)
    C = assembly.gradient_matrix(m)
    gptr = T(w, "grad_nodes_ptr")
    gn = T(w, "grad_nodes")
    for i, d in enumerate(dec.dofs):
        cols, _ = coarse.local_gradient_basis(C, d)
        assert np.array_equal(gn[gptr[i]:gptr[i + 1]], cols)


def test_bad_arguments_fail_loudly():
    from paper_2311_18783_b200 import topology_array as T
    from paper_2311_18783_b200._lib import MDDError
    w = workloads.custom(5, 4, 4, 2, 2, 2)   # 5 not divisible by 2
    with pytest.raises(MDDError):
        T(w, "sub_ptr")


def test_topology_bit_exact_c1_full_size():
    # BASELINE configs[1] at full size (220k free edges): numbering, the pattern
    # of A and every subdomain's dof list N_i agree bit-for-bit with the oracle
    from paper_2311_18783_b200 import topology_array as T
    w = workloads.make("c1")
    m = om.mesh_of(w)
    assert np.array_equal(T(w, "edge_tail"), m.edges[:, 0])
    assert np.array_equal(T(w, "edge_head"), m.edges[:, 1])
    assert np.array_equal(T(w, "free_edges"), m.free_edges)
    A, _, _ = assembly.system_matrix(m, w.mu_inv, w.eps, w.gamma)
    assert np.array_equal(T(w, "A_ptr"), A.indptr)
    assert np.array_equal(T(w, "A_idx"), A.indices)
    dec = dd.decompose(m, w.px, w.py, w.pz, w.overlap)
    ptr, dofs = T(w, "sub_ptr"), T(w, "sub_dofs")
    for i, d in enumerate(dec.dofs):
        assert np.array_equal(dofs[ptr[i]:ptr[i + 1]], d)


def test_null_handles_and_bad_values_return_errors():
    """Every entry point rejects null handles / pointers with MDD_ERR_ARG and a
    message, without touching a device (runs without a GPU)."""
    import ctypes as C
    from paper_2311_18783_b200 import _lib as L
    lib = L.lib()
    it, rel = C.c_int(0), C.c_double(0.0)
    assert lib.mdd_solve(None, None, None, 1e-8, 10, C.byref(it), C.byref(rel)) == L.MDD_ERR_ARG
    assert lib.mdd_last_error()
    assert lib.mdd_solve_host(None, None, None, 1e-8, 10, C.byref(it), C.byref(rel)) == L.MDD_ERR_ARG
    for fn in ("mdd_apply_preconditioner", "mdd_apply_operator", "mdd_apply_local", "mdd_apply_coarse"):
        assert getattr(lib, fn)(None, None, None) == L.MDD_ERR_ARG, fn
    assert lib.mdd_set_variant(None, 0) == L.MDD_ERR_ARG
    assert lib.mdd_set_stream(None, None) == L.MDD_ERR_ARG
    assert lib.mdd_setup(None, None) == L.MDD_ERR_ARG
    lib.mdd_destroy(None)   # a no-op
