"""ctypes binding of libmaxwell_dd.so (argument marshalling only).

Every numerical step runs inside the CUDA library; this module only converts
Python / numpy / torch arguments to the plain pointers and sizes declared in
include/maxwell_dd.h.  Importing it fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MDD_LIB_PATH: an experiment build of the same library (tools/, never the default)
LIB_PATH = os.environ.get("MDD_LIB_PATH") or os.path.join(HERE, "libmaxwell_dd.so")

MDD_OK, MDD_ERR_CUDA, MDD_ERR_ARG, MDD_ERR_NOTPD, MDD_ERR_NOCONV, MDD_ERR_INTERNAL, MDD_ERR_BREAKDOWN = range(7)
DIRICHLET = {"outer": 0, "all": 1, "none": 2}
COARSE = {"none": 0, "snk": 1, "nk": 2}
VARIANT = {"as2": 0, "additive": 1, "as1": 2, "as2_coarse_start": 3}

INFO_NAMES = ["n", "nedges", "nfree_nodes", "nsub", "nnz_A", "nloc", "grad_candidates",
              "grad_rank", "ngeneo", "n0", "local_factor_nnz", "coarse_factor_nnz",
              "local_supernodes", "local_levels", "coarse_supernodes", "coarse_levels",
              "nnz_Z", "kernels_per_iter", "last_launches",
              "coarse_perturbed", "nnz_Zg", "nnz_W",
              "local_sn_packed", "local_sn_strip", "local_sn_2d", "local_blocked_fronts",
              "coarse_sn_packed", "coarse_sn_strip", "coarse_sn_2d", "coarse_blocked_fronts",
              "geneo_lanczos"]
INT_ARRAYS = {"edge_tail": 0, "edge_head": 1, "free_edges": 2, "free_nodes": 3, "A_ptr": 4,
              "A_idx": 5, "sub_ptr": 6, "sub_dofs": 7, "grad_nodes_ptr": 8, "grad_nodes": 9,
              "geneo_count": 10, "E_ptr": 11, "E_idx": 12}
DBL_ARRAYS = {"A_val": 0, "K_val": 1, "M_val": 2, "geneo_lambda": 3, "setup_times": 4, "E_val": 5}
SHARD_ARRAYS = {"subs": 0, "owned": 1, "halo": 2, "send_ptr": 3, "send_idx": 4, "recv_ptr": 5, "recv_idx": 6,
                "dof_owner": 7}
PROF_NAMES = ["spmv", "local", "prec_other", "coarse", "vector", "total"]


class SetupDesc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("h", C.c_double),
                ("cube_mask", C.POINTER(C.c_uint8)), ("dirichlet", C.c_int),
                ("mu_inv", C.POINTER(C.c_double)), ("eps", C.POINTER(C.c_double)),
                ("gamma", C.c_double), ("px", C.c_int), ("py", C.c_int), ("pz", C.c_int),
                ("overlap", C.c_int), ("coarse_threshold", C.c_double), ("coarse_kind", C.c_int),
                ("variant", C.c_int), ("device", C.c_int), ("reserved", C.c_int * 8)]


# every symbol include/maxwell_dd.h declares (checked by tests/test_abi.py)
EXPORTS = ["mdd_setup", "mdd_destroy", "mdd_solve", "mdd_solve_host", "mdd_set_stream", "mdd_set_variant",
           "mdd_apply_preconditioner",
           "mdd_apply_operator", "mdd_apply_local", "mdd_apply_coarse", "mdd_apply_local_parts",
           "mdd_apply_coarse_inverse", "mdd_shard_setup", "mdd_shard_info", "mdd_shard_nccl_init",
           "mdd_shard_solve", "mdd_shard_solve_group", "mdd_info",
           "mdd_get_int_array", "mdd_topology_int_array", "mdd_shard_int_array", "mdd_tree_split",
           "mdd_get_double_array",
           "mdd_phase_name", "mdd_set_profiling", "mdd_sweep_timing", "mdd_profile", "mdd_last_error"]


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2311_18783_b200.build` "
                          "(the CUDA library is required; there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    dp = C.POINTER(C.c_double)
    lp = C.POINTER(C.c_int64)
    sig = {
        "mdd_setup": (C.c_int, [C.POINTER(SetupDesc), C.POINTER(P)]),
        "mdd_destroy": (None, [P]),
        "mdd_solve": (C.c_int, [P, P, P, C.c_double, C.c_int, C.POINTER(C.c_int), dp]),
        "mdd_solve_host": (C.c_int, [P, dp, dp, C.c_double, C.c_int, C.POINTER(C.c_int), dp]),
        "mdd_set_stream": (C.c_int, [P, P]),
        "mdd_set_variant": (C.c_int, [P, C.c_int]),
        "mdd_apply_preconditioner": (C.c_int, [P, P, P]),
        "mdd_apply_operator": (C.c_int, [P, P, P]),
        "mdd_apply_local": (C.c_int, [P, P, P]),
        "mdd_apply_coarse": (C.c_int, [P, P, P]),
        "mdd_apply_local_parts": (C.c_int, [P, P, P]),
        "mdd_apply_coarse_inverse": (C.c_int, [P, P, P]),
        "mdd_shard_setup": (C.c_int, [P, C.c_int, C.c_int]),
        "mdd_shard_info": (C.c_int, [P, lp, C.c_int]),
        "mdd_shard_nccl_init": (C.c_int, [P, C.c_char_p, C.c_int, C.c_int]),
        "mdd_shard_solve": (C.c_int, [P, P, P, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_int), dp]),
        "mdd_shard_solve_group": (C.c_int, [C.POINTER(P), C.c_int, C.POINTER(P), C.POINTER(P), C.c_double,
                                            C.c_int, C.POINTER(C.c_int), dp]),
        "mdd_info": (C.c_int, [P, lp, C.c_int]),
        "mdd_get_int_array": (C.c_int, [P, C.c_int, lp, C.c_int64, lp]),
        "mdd_topology_int_array": (C.c_int, [C.POINTER(SetupDesc), C.c_int, lp, C.c_int64, lp]),
        "mdd_shard_int_array": (C.c_int, [C.POINTER(SetupDesc), C.c_int, C.c_int, C.c_int, lp, C.c_int64, lp]),
        "mdd_tree_split": (C.c_int, [C.c_int, C.POINTER(C.c_int32), lp, C.c_int, C.POINTER(C.c_int32)]),
        "mdd_get_double_array": (C.c_int, [P, C.c_int, dp, C.c_int64, lp]),
        "mdd_phase_name": (C.c_char_p, [C.c_int]),
        "mdd_set_profiling": (C.c_int, [P, C.c_int]),
        "mdd_profile": (C.c_int, [P, dp, lp, C.c_int]),
        "mdd_sweep_timing": (C.c_int, [P, C.c_int, dp, lp]),
        "mdd_last_error": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


class MDDError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"maxwell_dd error {code}: {msg}")
        self.code = code


def check(rc: int):
    if rc != MDD_OK:
        raise MDDError(rc, lib().mdd_last_error().decode())
