"""ctypes binding of libamg_b200.so — argument marshalling only.

Every step of the solve path runs in the library's CUDA kernels; this module never computes any
part of the method.  If the shared library is missing the import fails loudly (no fallback).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# AMG_LIB=checked loads the checked build (device-side invariant checks, build.py --checked)
LIB_PATH = os.path.join(HERE, "libamg_b200_checked.so" if os.environ.get("AMG_LIB") == "checked" else "libamg_b200.so")

AMG_OK, AMG_NOT_CONVERGED = 0, 1
STATUS = {0: "AMG_OK", 1: "AMG_NOT_CONVERGED", -1: "AMG_EINVAL", -2: "AMG_ENOMEM", -3: "AMG_ECUDA",
          -4: "AMG_ENCCL", -5: "AMG_ENOTSPD", -6: "AMG_ENODEV"}

# every symbol declared in include/amg_b200.h
EXPORTED = ["amg_iga_poisson", "amg_iga_tables", "amg_csr_free", "amg_free", "amg_params_default",
            "amg_set_allocator", "amg_setup", "amg_setup_take", "amg_pcg_solve", "amg_pcg_solve_host", "amg_vcycle",
            "amg_level_apply", "amg_hierarchy_info", "amg_hierarchy_export", "amg_set_profiling",
            "amg_get_kernel_stats", "amg_operator_config", "amg_operator_set_config", "amg_get_level_times", "amg_nccl_unique_id", "amg_local_rows",
            "amg_dist_view_get", "amg_share_export", "amg_setup_from_share", "amg_setup_from_share_take",
            "amg_malloc", "amg_set_num_threads",
            "amg_hierarchy_free",
            "amg_last_error"]


class AmgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class amg_csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_double))]


class amg_iga_desc(C.Structure):
    _fields_ = [("dim", C.c_int), ("degree", C.c_int), ("n_elem", C.c_int), ("dirichlet_sides", C.c_uint32),
                ("rhs", C.c_int), ("geometry", C.c_int)]


class amg_params(C.Structure):
    _fields_ = [("agg_steps", C.c_int), ("smooth_prolong", C.c_int), ("match_threshold", C.c_double),
                ("filter_theta", C.c_double), ("cheb_degree", C.c_int), ("coarse_sweeps", C.c_int),
                ("coarse_size", C.c_int64), ("max_levels", C.c_int), ("format", C.c_int),
                ("host_only", C.c_int), ("num_threads", C.c_int), ("krylov", C.c_int), ("coarse_solver", C.c_int),
                ("coarse_tol", C.c_double), ("coarse_maxit", C.c_int)]


class amg_dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("nccl_id", C.c_ubyte * 128), ("device", C.c_int)]


class amg_kernel_stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("total_ms", C.c_double), ("bytes_per_launch", C.c_double),
                ("kernels_launched", C.c_int64)]


class amg_op_config(C.Structure):
    _fields_ = [("layout", C.c_int), ("kernel", C.c_int), ("G", C.c_int), ("U", C.c_int), ("stored", C.c_int64),
                ("tuned_us", C.c_double), ("alg_bytes", C.c_double), ("nnz", C.c_int64), ("n_values", C.c_int64),
                ("value_index_bytes", C.c_int), ("sellvi_parts", C.c_int), ("offset_bits", C.c_int)]


class amg_dist_view(C.Structure):
    _fields_ = [("nranks", C.c_int), ("replicated", C.c_int), ("full_cols", C.c_int),
                ("row_begin", C.c_int64), ("row_end", C.c_int64), ("col_begin", C.c_int64), ("col_end", C.c_int64),
                ("n_ghost", C.c_int64), ("n_ghost_lo", C.c_int64), ("ghost", C.POINTER(C.c_int64)),
                ("send_count", C.POINTER(C.c_int32)), ("send_off", C.POINTER(C.c_int32)),
                ("send_idx", C.POINTER(C.c_int32)), ("recv_count", C.POINTER(C.c_int32)),
                ("recv_off", C.POINTER(C.c_int32)), ("local", amg_csr)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2511_21268_b200.build` "
                          "(there is no CPU fallback)")
    try:  # load torch first so the library binds to the process's single libnccl.so.2 (torch's)
        import torch  # noqa: F401
    except Exception:  # noqa: BLE001
        pass
    L = C.CDLL(LIB_PATH)
    vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
    P = C.POINTER
    sig = {
        "amg_iga_poisson": ([P(amg_iga_desc), P(P(amg_csr)), P(dp)], C.c_int),
        "amg_iga_tables": ([C.c_int, C.c_int, dp, dp], C.c_int),
        "amg_csr_free": ([P(amg_csr)], None),
        "amg_free": ([vp], None),
        "amg_params_default": ([P(amg_params), C.c_int], C.c_int),
        "amg_set_allocator": ([vp, vp], C.c_int),
        "amg_setup": ([P(amg_csr), P(amg_params), P(amg_dist), P(vp)], C.c_int),
        "amg_setup_take": ([P(amg_csr), P(amg_params), P(amg_dist), P(vp)], C.c_int),
        "amg_pcg_solve": ([vp, vp, vp, C.c_double, C.c_int, vp, ip, dp, dp], C.c_int),
        "amg_pcg_solve_host": ([vp, dp, dp, C.c_double, C.c_int, vp, ip, dp, dp], C.c_int),
        "amg_vcycle": ([vp, vp, vp, vp], C.c_int),
        "amg_level_apply": ([vp, C.c_int, C.c_int, vp, vp, vp], C.c_int),
        "amg_hierarchy_info": ([vp, P(C.c_int64), P(C.c_int64), P(C.c_int64), P(C.c_int64), dp], C.c_int),
        "amg_hierarchy_export": ([vp, C.c_int, P(P(amg_csr)), P(P(amg_csr)), P(P(C.c_int32)), P(dp), dp], C.c_int),
        "amg_set_profiling": ([vp, C.c_int], C.c_int),
        "amg_get_kernel_stats": ([vp, P(amg_kernel_stats)], C.c_int),
        "amg_operator_config": ([vp, C.c_int, C.c_int, P(amg_op_config)], C.c_int),
        "amg_operator_set_config": ([vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int], C.c_int),
        "amg_get_level_times": ([vp, P(C.c_double), C.c_int, P(C.c_int)], C.c_int),
        "amg_nccl_unique_id": ([P(C.c_ubyte)], C.c_int),
        "amg_local_rows": ([vp, P(C.c_int64), P(C.c_int64)], C.c_int),
        "amg_dist_view_get": ([vp, C.c_int, C.c_int, P(amg_dist_view)], C.c_int),
        "amg_share_export": ([vp, C.c_int, C.c_int, P(vp), P(C.c_int64)], C.c_int),
        "amg_setup_from_share": ([vp, C.c_int64, P(amg_dist), C.c_int, P(vp)], C.c_int),
        "amg_setup_from_share_take": ([vp, C.c_int64, P(amg_dist), C.c_int, P(vp)], C.c_int),
        "amg_malloc": ([C.c_int64], vp),
        "amg_set_num_threads": ([C.c_int], C.c_int),
        "amg_hierarchy_free": ([vp], None),
        "amg_last_error": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def check(status: int) -> int:
    if status not in (AMG_OK, AMG_NOT_CONVERGED):
        raise AmgError(status, lib().amg_last_error().decode())
    return status


def csr_to_numpy(c: amg_csr):
    """Copy a library-owned amg_csr into numpy arrays (indptr, indices, data, shape)."""
    n, nnz = c.n_rows, c.nnz
    rp = np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)).copy()
    ci = np.ctypeslib.as_array(c.col, shape=(max(nnz, 1),))[:nnz].copy()
    v = np.ctypeslib.as_array(c.val, shape=(max(nnz, 1),))[:nnz].copy()
    return rp, ci, v, (n, c.n_cols)
