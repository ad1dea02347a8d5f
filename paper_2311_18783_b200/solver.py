"""Thin Python front end of the C ABI (argument marshalling only)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def _desc(w, coarse="snk", variant="as2", device=0, geneo=True) -> tuple:
    mask = np.ascontiguousarray(w.cube_mask, dtype=np.uint8)
    mu = np.ascontiguousarray(w.mu_inv, dtype=np.float64)
    ep = np.ascontiguousarray(w.eps, dtype=np.float64)
    d = L.SetupDesc()
    d.nx, d.ny, d.nz, d.h = w.nx, w.ny, w.nz, float(w.h)
    d.cube_mask = mask.ctypes.data_as(C.POINTER(C.c_uint8))
    d.dirichlet = L.DIRICHLET[w.dirichlet]
    d.mu_inv = mu.ctypes.data_as(C.POINTER(C.c_double))
    d.eps = ep.ctypes.data_as(C.POINTER(C.c_double))
    d.gamma = float(w.gamma)
    d.px, d.py, d.pz, d.overlap = w.px, w.py, w.pz, w.overlap
    d.coarse_threshold = float(w.threshold) if geneo else 0.0
    d.coarse_kind = L.COARSE[coarse]
    d.variant = L.VARIANT[variant]
    d.device = device
    return d, (mask, mu, ep)


def topology_array(w, name: str) -> np.ndarray:
    """Host-only integer topology (numbering, pattern of A, N_i, G_i columns)."""
    d, keep = _desc(w)
    n = C.c_int64(0)
    which = L.INT_ARRAYS[name]
    L.check(L.lib().mdd_topology_int_array(C.byref(d), which, None, 0, C.byref(n)))
    out = np.empty(n.value, np.int64)
    L.check(L.lib().mdd_topology_int_array(C.byref(d), which,
                                           out.ctypes.data_as(C.POINTER(C.c_int64)), n.value,
                                           C.byref(n)))
    return out


def shard_array(w, rank: int, nranks: int, name: str) -> np.ndarray:
    """Host-only sharded-solve plan of `rank` (mdd_shard_int_array)."""
    d, keep = _desc(w)
    n = C.c_int64(0)
    which = L.SHARD_ARRAYS[name]
    L.check(L.lib().mdd_shard_int_array(C.byref(d), rank, nranks, which, None, 0, C.byref(n)))
    out = np.empty(n.value, np.int64)
    L.check(L.lib().mdd_shard_int_array(C.byref(d), rank, nranks, which,
                                        out.ctypes.data_as(C.POINTER(C.c_int64)), n.value, C.byref(n)))
    return out


def tree_split(parent, cost, nranks: int) -> np.ndarray:
    """Host-only subtree-to-rank mapping of a supernode tree (mdd_tree_split):
    -1 = replicated top supernode, else the rank sweeping it with its subtree."""
    par = np.ascontiguousarray(parent, dtype=np.int32)
    cst = np.ascontiguousarray(cost, dtype=np.int64)
    if par.shape != cst.shape or par.ndim != 1:
        raise ValueError("parent and cost must be 1-D arrays of equal length")
    out = np.empty(len(par), np.int32)
    L.check(L.lib().mdd_tree_split(len(par), par.ctypes.data_as(C.POINTER(C.c_int32)),
                                   cst.ctypes.data_as(C.POINTER(C.c_int64)), int(nranks),
                                   out.ctypes.data_as(C.POINTER(C.c_int32))))
    return out


def _ptr(t, n=None, device=None) -> int:
    """Device pointer of a contiguous float64 CUDA tensor of n elements on the
    handle's device (the C ABI reads / writes exactly n doubles)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
            and t.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    if device is not None and t.device.index != device:
        raise ValueError(f"tensor on cuda:{t.device.index}, handle on cuda:{device}")
    return t.data_ptr()


def _host(a, n, name):
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
            and a.size == n):
        raise ValueError(f"{name}: expected a C-contiguous float64 array of {n} elements")
    return a


class MaxwellDD:
    """Handle of one set-up problem: ``MaxwellDD(workload)`` runs the device setup;
    ``solve(f)`` runs PCG on the device."""

    def __init__(self, w, coarse="snk", variant="as2", device=0, geneo=True):
        self.w = w
        self.variant = variant
        self.device = device
        d, keep = _desc(w, coarse, variant, device, geneo)
        h = C.c_void_p()
        L.check(L.lib().mdd_setup(C.byref(d), C.byref(h)))
        self._h = h
        self.info = self._info()
        self.n = int(self.info["n"])

    def close(self):
        if getattr(self, "_h", None):
            L.lib().mdd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _info(self):
        out = (C.c_int64 * len(L.INFO_NAMES))()
        L.check(L.lib().mdd_info(self._h, out, len(L.INFO_NAMES)))
        return dict(zip(L.INFO_NAMES, list(out)))

    def int_array(self, name):
        n = C.c_int64(0)
        which = L.INT_ARRAYS[name]
        L.check(L.lib().mdd_get_int_array(self._h, which, None, 0, C.byref(n)))
        out = np.empty(n.value, np.int64)
        L.check(L.lib().mdd_get_int_array(self._h, which, out.ctypes.data_as(C.POINTER(C.c_int64)),
                                          n.value, C.byref(n)))
        return out

    def double_array(self, name):
        n = C.c_int64(0)
        which = L.DBL_ARRAYS[name]
        L.check(L.lib().mdd_get_double_array(self._h, which, None, 0, C.byref(n)))
        out = np.empty(n.value, np.float64)
        L.check(L.lib().mdd_get_double_array(self._h, which, out.ctypes.data_as(C.POINTER(C.c_double)),
                                             n.value, C.byref(n)))
        return out

    def setup_times(self):
        t = self.double_array("setup_times")
        return {L.lib().mdd_phase_name(k).decode(): float(v) for k, v in enumerate(t)}

    # ------------------------------------------------------------- device ops
    def solve(self, f, x, tol=1e-8, maxit=1000):
        it = C.c_int(0)
        rel = C.c_double(0.0)
        rc = L.lib().mdd_solve(self._h, self._p(f), self._p(x), tol, maxit, C.byref(it), C.byref(rel))
        if rc not in (L.MDD_OK, L.MDD_ERR_NOCONV):
            L.check(rc)
        return it.value, rel.value, rc == L.MDD_OK

    def _p(self, t, n=None):
        return _ptr(t, self.n if n is None else n, self.device)

    def solve_host(self, f: np.ndarray, tol=1e-8, maxit=1000):
        f = _host(np.ascontiguousarray(f, dtype=np.float64), self.n, "f")
        x = np.empty_like(f)
        it = C.c_int(0)
        rel = C.c_double(0.0)
        dp = C.POINTER(C.c_double)
        rc = L.lib().mdd_solve_host(self._h, f.ctypes.data_as(dp), x.ctypes.data_as(dp), tol, maxit,
                                    C.byref(it), C.byref(rel))
        if rc not in (L.MDD_OK, L.MDD_ERR_NOCONV):
            L.check(rc)
        return x, it.value, rel.value

    def set_stream(self, stream):
        """Run the handle's device work on a torch.cuda.Stream (or raw handle int);
        None restores the library's private stream."""
        raw = None if stream is None else int(getattr(stream, "cuda_stream", stream))
        L.check(L.lib().mdd_set_stream(self._h, raw))

    def set_variant(self, variant: str):
        """Switch the preconditioner variant ("as2", "as2_coarse_start",
        "additive", "as1") without redoing the setup."""
        L.check(L.lib().mdd_set_variant(self._h, L.VARIANT[variant]))
        self.variant = variant

    def last_launches(self):
        return int(self._info()["last_launches"])

    def solve_host_into(self, f: np.ndarray, x: np.ndarray, tol=1e-8, maxit=1000):
        """mdd_solve_host on caller-owned (e.g. pinned) float64 host arrays."""
        _host(f, self.n, "f")
        _host(x, self.n, "x")
        it = C.c_int(0)
        rel = C.c_double(0.0)
        dp = C.POINTER(C.c_double)
        rc = L.lib().mdd_solve_host(self._h, f.ctypes.data_as(dp), x.ctypes.data_as(dp), tol, maxit,
                                    C.byref(it), C.byref(rel))
        if rc not in (L.MDD_OK, L.MDD_ERR_NOCONV):
            L.check(rc)
        return x, it.value, rel.value

    def bytes_model(self):
        """Algorithmic HBM bytes of the solve-phase operations:
        every stored value / index the operation needs, read once, and every
        output written once."""
        i = self.info
        n, nnzA, nloc = i["n"], i["nnz_A"], i["nloc"]
        spmv = 12 * nnzA + 8 * (n + 1) + 16 * n
        # local sweep: every factor entry once per direction, D^{-1}, the restriction
        # of r and the prolongated result (the kernel's own scratch is not counted)
        local = 2 * 8 * i["local_factor_nnz"] + 8 * nloc + 8 * n + 8 * n
        # coarse: gradient part of Z as CSR (12 B / entry) and the dense GenEO blocks
        # (8 B / entry), each read in Z^T v and in Z y; E's factor in both sweeps
        coarse = (2 * 12 * i["nnz_Zg"] + 2 * 8 * i["nnz_W"] + 2 * 8 * i["coarse_factor_nnz"]
                  + 8 * i["n0"] + 16 * n) if i["n0"] else 0
        vec = 8 * n * 4
        precond = local + 2 * coarse + 2 * spmv + vec
        # the PCG loop's preconditioner: with the coarse start (reading R13) one
        # coarse correction and one A product, w + Q (r - A w)
        loop = local + coarse + spmv + 8 * n * 5 if getattr(self, "variant", "as2") == "as2_coarse_start" \
            else precond
        return {"spmv": spmv, "local": local, "coarse": coarse, "precond": precond,
                "precond_in_loop": loop, "iteration": loop + spmv + 8 * n * 7}

    def apply_preconditioner(self, r, z):
        L.check(L.lib().mdd_apply_preconditioner(self._h, self._p(r), self._p(z)))

    def apply_operator(self, x, y):
        L.check(L.lib().mdd_apply_operator(self._h, self._p(x), self._p(y)))

    def apply_local(self, r, z):
        L.check(L.lib().mdd_apply_local(self._h, self._p(r), self._p(z)))

    def apply_coarse(self, v, y):
        L.check(L.lib().mdd_apply_coarse(self._h, self._p(v), self._p(y)))

    # ------------------------------------------------ parity diagnostics
    def apply_local_parts(self, r, xloc):
        """xloc = concatenated A_i^{-1} R_i r (subdomain-major, N_i order)."""
        L.check(L.lib().mdd_apply_local_parts(self._h, self._p(r), self._p(xloc, int(self.info["nloc"]))))

    def apply_coarse_inverse(self, v, y):
        """y = E^{-1} v for the factorised E, coarse-position order."""
        n0 = int(self.info["n0"])
        L.check(L.lib().mdd_apply_coarse_inverse(self._h, self._p(v, n0), self._p(y, n0)))

    def coarse_matrix(self):
        """The factorised (Jacobi-scaled) E as a scipy CSR matrix, coarse-position order."""
        import scipy.sparse as sp
        n0 = int(self.info["n0"])
        return sp.csr_matrix((self.double_array("E_val"), self.int_array("E_idx"), self.int_array("E_ptr")),
                             shape=(n0, n0))

    # ------------------------------------------------------ sharded solve
    def shard_setup(self, rank: int, nranks: int):
        """This handle becomes rank `rank` of a sharded solve (mdd_shard_setup)."""
        L.check(L.lib().mdd_shard_setup(self._h, rank, nranks))
        out = (C.c_int64 * 8)()
        L.check(L.lib().mdd_shard_info(self._h, out, 8))
        self.shard = {"rank": rank, "nranks": nranks, "n_own": int(out[0]), "n_local": int(out[1]),
                      "subdomains": int(out[2]), "factor_nnz": int(out[3]), "coarse_distributed": bool(out[4]),
                      "coarse_swept_nnz": int(out[5]), "coarse_top_nnz": int(out[6]),
                      "coarse_exchange": int(out[7])}
        self.owned = shard_array(self.w, rank, nranks, "owned")
        return self.shard

    def shard_nccl_init(self, unique_id: bytes):
        """NCCL communicator of the ranks (unique_id: 128 bytes from rank 0)."""
        L.check(L.lib().mdd_shard_nccl_init(self._h, bytes(unique_id), self.shard["rank"], self.shard["nranks"]))

    def shard_solve(self, f_own, x_own, tol=1e-8, maxit=1000):
        """This rank's part of the sharded PCG (collective over the ranks); f_own /
        x_own: n_own float64 CUDA tensors on this rank's owned dofs."""
        n = self.shard["n_own"]
        it = C.c_int(0)
        rel = C.c_double(0.0)
        rc = L.lib().mdd_shard_solve(self._h, self._p(f_own, n), self._p(x_own, n), tol, maxit, 0,
                                     C.byref(it), C.byref(rel))
        if rc not in (L.MDD_OK, L.MDD_ERR_NOCONV):
            L.check(rc)
        return it.value, rel.value, rc == L.MDD_OK

    def set_profiling(self, on=True):
        L.check(L.lib().mdd_set_profiling(self._h, 1 if on else 0))

    def sweep_timing(self, which="local"):
        """(total device ms, launches) of the persistent sweep kernel so far."""
        ms = C.c_double(0.0)
        n = C.c_int64(0)
        L.check(L.lib().mdd_sweep_timing(self._h, 0 if which == "local" else 1, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def profile(self):
        ms = (C.c_double * len(L.PROF_NAMES))()
        ln = (C.c_int64 * len(L.PROF_NAMES))()
        L.check(L.lib().mdd_profile(self._h, ms, ln, len(L.PROF_NAMES)))
        return {k: (ms[i], ln[i]) for i, k in enumerate(L.PROF_NAMES)}


def shard_solve_group(handles, f_own, x_own, tol=1e-8, maxit=1000):
    """Sharded PCG of several handles of this process on one GPU (handle k = rank
    k), exchanging through device copies (mdd_shard_solve_group)."""
    k = len(handles)
    P = C.c_void_p
    hs = (P * k)(*[h._h.value for h in handles])
    fs = (P * k)(*[h._p(f, h.shard["n_own"]) for h, f in zip(handles, f_own)])
    xs = (P * k)(*[h._p(x, h.shard["n_own"]) for h, x in zip(handles, x_own)])
    it = C.c_int(0)
    rel = C.c_double(0.0)
    rc = L.lib().mdd_shard_solve_group(hs, k, fs, xs, tol, maxit, C.byref(it), C.byref(rel))
    if rc not in (L.MDD_OK, L.MDD_ERR_NOCONV):
        L.check(rc)
    return it.value, rel.value, rc == L.MDD_OK
