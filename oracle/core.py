"""ctypes wrapper around oracle.c (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from . import tables

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "_build", "liboracle.so")


def build_liboracle(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2 -ffp-contract=off: no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_SO), exist_ok=True)
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class _CSR(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("rp", C.POINTER(C.c_int64)), ("ci", C.POINTER(C.c_int32)), ("v", C.POINTER(C.c_double))]


class _Params(C.Structure):
    _fields_ = [("agg_steps", C.c_int), ("smooth_prolong", C.c_int), ("match_threshold", C.c_double),
                ("filter_theta", C.c_double), ("cheb_degree", C.c_int), ("coarse_sweeps", C.c_int),
                ("coarse_size", C.c_int64), ("max_levels", C.c_int), ("coarse_solver", C.c_int),
                ("coarse_tol", C.c_double), ("coarse_maxit", C.c_int), ("tie_break", C.c_int),
                ("omega_norm", C.c_int)]


class _Level(C.Structure):
    _fields_ = [("N", C.c_int64), ("K", _CSR), ("P", _CSR), ("R", _CSR),
                ("agg", C.POINTER(C.c_int32)), ("ptent", C.POINTER(C.c_double)),
                ("dhat", C.POINTER(C.c_double)), ("w", C.POINTER(C.c_double)), ("omega", C.c_double)]


_lib = None
ITER_CB = C.CFUNCTYPE(C.c_int, C.c_int, C.c_void_p)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build_liboracle())
        dp = C.POINTER(C.c_double)
        L.or_assemble.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, C.POINTER(_CSR)]
        L.or_spmv.argtypes = [C.POINTER(_CSR), dp, dp]
        L.or_setup.argtypes = [C.POINTER(_CSR), C.POINTER(_Params), C.POINTER(C.c_void_p)]
        L.or_hier_free.argtypes = [C.c_void_p]
        L.or_hier_nlevels.argtypes = [C.c_void_p]
        L.or_hier_level.argtypes = [C.c_void_p, C.c_int]
        L.or_hier_level.restype = C.POINTER(_Level)
        L.or_vcycle.argtypes = [C.c_void_p, dp, dp]
        L.or_smooth.argtypes = [C.c_void_p, C.c_int, dp, dp, C.c_int]
        L.or_pcg.argtypes = [C.c_void_p, dp, dp, C.c_double, C.c_int, C.POINTER(C.c_int), dp, dp]
        L.or_fcg.argtypes = [C.c_void_p, dp, dp, C.c_double, C.c_int, C.POINTER(C.c_int), dp, dp]
        L.or_fcg_cb.argtypes = [C.c_void_p, dp, dp, C.c_double, C.c_int, C.POINTER(C.c_int), dp, dp, ITER_CB,
                                C.c_void_p]
        L.or_cij.argtypes = [C.c_double] * 5
        L.or_cij.restype = C.c_double
        L.or_pairwise.argtypes = [C.POINTER(_CSR), dp, C.c_double, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), dp, dp]
        L.or_pairwise.restype = C.c_int64
        L.or_galerkin_pairwise.argtypes = [C.POINTER(_CSR), C.POINTER(C.c_int32), dp, C.c_int64, C.POINTER(_CSR)]
        L.or_csr_new.restype = C.POINTER(_CSR)
        L.or_csr_delete.argtypes = [C.POINTER(_CSR)]
        _lib = L
    return _lib


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _csr_to_scipy(c: _CSR) -> sp.csr_matrix:
    n, m, nnz = c.nrows, c.ncols, c.nnz
    if n == 0:
        return sp.csr_matrix((0, m))
    rp = np.ctypeslib.as_array(c.rp, shape=(n + 1,)).copy()
    ci = np.ctypeslib.as_array(c.ci, shape=(max(nnz, 1),))[:nnz].copy()
    v = np.ctypeslib.as_array(c.v, shape=(max(nnz, 1),))[:nnz].copy()
    A = sp.csr_matrix((v, ci, rp), shape=(n, m))
    A.has_sorted_indices = True
    return A


class _Borrowed:
    """A scipy CSR viewed as an ocsr (arrays kept alive by this object)."""

    def __init__(self, A: sp.csr_matrix):
        A = sp.csr_matrix(A)
        A.sort_indices()
        self.rp = np.ascontiguousarray(A.indptr, dtype=np.int64)
        self.ci = np.ascontiguousarray(A.indices, dtype=np.int32)
        self.v = np.ascontiguousarray(A.data, dtype=np.float64)
        self.c = _CSR(A.shape[0], A.shape[1], A.nnz, self.rp.ctypes.data_as(C.POINTER(C.c_int64)),
                      self.ci.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(self.v))


def assemble(dim: int, p: int, n: int, dirichlet_sides: int = 0b000111) -> sp.csr_matrix:
    """c.4: stiffness K of the free DOFs by the Kronecker sum of the exact 1-D tables."""
    Mb, Kb = tables.banded_tables(p, n)
    Mb = np.ascontiguousarray(Mb)
    Kb = np.ascontiguousarray(Kb)
    out = lib().or_csr_new()
    rc = lib().or_assemble(dim, p, n, dirichlet_sides, _dptr(Mb), _dptr(Kb), out)
    if rc:
        raise RuntimeError(f"or_assemble failed: {rc}")
    A = _csr_to_scipy(out.contents)
    lib().or_csr_delete(out)
    return A


def spmv(A: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    b = _Borrowed(A)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.shape[0])
    lib().or_spmv(C.byref(b.c), _dptr(x), _dptr(y))
    return y


def cij(kij, kii, kjj, wi, wj) -> float:
    """eq:cij for the ordered pair i<j, in the c.7 evaluation order."""
    return lib().or_cij(kij, kii, kjj, wi, wj)


def pairwise(A: sp.csr_matrix, w: np.ndarray, threshold: float = 1.0):
    """One pairwise matching/aggregation step (c.7-c.9) → (mate, agg, pvals, w_coarse)."""
    b = _Borrowed(A)
    n = A.shape[0]
    w = np.ascontiguousarray(w, dtype=np.float64)
    mate = np.empty(n, np.int32)
    agg = np.empty(n, np.int32)
    pv = np.empty(n)
    wn = np.empty(max(n, 1))
    nc = lib().or_pairwise(C.byref(b.c), _dptr(w), threshold, mate.ctypes.data_as(C.POINTER(C.c_int32)),
                           agg.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(pv), _dptr(wn))
    if nc < 0:
        raise RuntimeError(f"or_pairwise failed: {nc}")
    return mate, agg, pv, wn[:nc].copy()


def galerkin_pairwise(A: sp.csr_matrix, agg: np.ndarray, pv: np.ndarray, nc: int) -> sp.csr_matrix:
    """c.10: the intermediate Galerkin operator sym(P_sᵀ A P_s) of one pairwise step."""
    b = _Borrowed(A)
    agg = np.ascontiguousarray(agg, dtype=np.int32)
    pv = np.ascontiguousarray(pv, dtype=np.float64)
    out = lib().or_csr_new()
    rc = lib().or_galerkin_pairwise(C.byref(b.c), agg.ctypes.data_as(C.POINTER(C.c_int32)), _dptr(pv), nc, out)
    if rc:
        raise RuntimeError(f"or_galerkin_pairwise failed: {rc}")
    Ac = _csr_to_scipy(out.contents)
    lib().or_csr_delete(out)
    return Ac


@dataclass
class OParams:
    agg_steps: int = 3
    smooth_prolong: int = 1
    match_threshold: float = 1.0
    filter_theta: float = 0.01
    cheb_degree: int = 8
    coarse_sweeps: int = 30
    coarse_size: int = 50
    max_levels: int = 20
    coarse_solver: int = 0      # 0: ℓ1-Jacobi sweeps (§4, c.17); 1: diagonal-PCG to coarse_tol (§5.1)
    coarse_tol: float = 1e-4
    coarse_maxit: int = 30
    tie_break: int = 0          # study knobs (oracle/scripts/opc_study.py); 0 = the canonical reading
    omega_norm: int = 0

    @staticmethod
    def for_degree(p: int, **kw) -> "OParams":
        from amg_inputs import CHEB_DEGREE
        return OParams(cheb_degree=CHEB_DEGREE[p], **kw)


@dataclass
class OLevel:
    N: int
    K: sp.csr_matrix
    P: sp.csr_matrix | None
    R: sp.csr_matrix | None
    agg: np.ndarray | None
    ptent: np.ndarray | None
    dhat: np.ndarray
    w: np.ndarray
    omega: float


class OHierarchy:
    def __init__(self, handle, prm: OParams):
        self._h = handle
        self.prm = prm
        L = lib()
        self.levels: list[OLevel] = []
        nl = L.or_hier_nlevels(handle)
        for l in range(nl):
            lv = L.or_hier_level(handle, l).contents
            N = lv.N
            last = l == nl - 1
            arr = lambda p_, n_, dt: np.ctypeslib.as_array(p_, shape=(max(n_, 1),))[:n_].copy()  # noqa: E731
            self.levels.append(OLevel(
                N=N, K=_csr_to_scipy(lv.K),
                P=None if last else _csr_to_scipy(lv.P), R=None if last else _csr_to_scipy(lv.R),
                agg=None if last else arr(lv.agg, N, np.int32),
                ptent=None if last else arr(lv.ptent, N, np.float64),
                dhat=arr(lv.dhat, N, np.float64), w=arr(lv.w, N, np.float64),
                omega=lv.omega if not last else 0.0))

    @property
    def nlevels(self) -> int:
        return len(self.levels)

    def opc(self) -> float:
        return sum(L.K.nnz for L in self.levels) / self.levels[0].K.nnz

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_hier_free(self._h)
            self._h = None


def setup(K: sp.csr_matrix, prm: OParams | None = None) -> OHierarchy:
    """c.6-c.15: the AMG hierarchy of K."""
    prm = prm or OParams()
    b = _Borrowed(K)
    cp = _Params(prm.agg_steps, prm.smooth_prolong, prm.match_threshold, prm.filter_theta,
                 prm.cheb_degree, prm.coarse_sweeps, prm.coarse_size, prm.max_levels,
                 prm.coarse_solver, prm.coarse_tol, prm.coarse_maxit, prm.tie_break, prm.omega_norm)
    h = C.c_void_p()
    rc = lib().or_setup(C.byref(b.c), C.byref(cp), C.byref(h))
    if rc:
        raise RuntimeError(f"or_setup failed: {rc}")
    return OHierarchy(h, prm)


def vcycle(H: OHierarchy, b: np.ndarray) -> np.ndarray:
    """c.18: one V-cycle application x = V(b)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    lib().or_vcycle(H._h, _dptr(b), _dptr(x))
    return x


def smooth(H: OHierarchy, level: int, b: np.ndarray, x0: np.ndarray | None = None) -> np.ndarray:
    """c.16: one application of the Chebyshev-ℓ1-Jacobi smoother on ``level`` (x0 = 0 if None)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    lib().or_smooth(H._h, level, _dptr(b), _dptr(x), 1 if x0 is None else 0)
    return x


def pcg(H: OHierarchy, F: np.ndarray, rtol: float = 1e-6, maxit: int = 200, u0: np.ndarray | None = None):
    """c.19: PCG → (u, iters, relres, history, status)."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    u = np.zeros_like(F) if u0 is None else np.array(u0, dtype=np.float64)
    it = C.c_int(0)
    rr = C.c_double(0.0)
    hist = np.full(maxit + 1, np.nan)
    rc = lib().or_pcg(H._h, _dptr(F), _dptr(u), rtol, maxit, C.byref(it), C.byref(rr), _dptr(hist))
    return u, it.value, rr.value, hist[: it.value + 1], rc


def fcg(H: OHierarchy, F: np.ndarray, rtol: float = 1e-6, maxit: int = 200, u0: np.ndarray | None = None,
        observer=None):
    """Flexible CG, Notay's FCG(1) → (u, iters, relres, history, status).
    observer(k) -> bool, if given, is called after iteration k (timing only); True stops the solve."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    u = np.zeros_like(F) if u0 is None else np.array(u0, dtype=np.float64)
    it = C.c_int(0)
    rr = C.c_double(0.0)
    hist = np.full(maxit + 1, np.nan)
    if observer is None:
        rc = lib().or_fcg(H._h, _dptr(F), _dptr(u), rtol, maxit, C.byref(it), C.byref(rr), _dptr(hist))
    else:
        cb = ITER_CB(lambda k, _ctx: 1 if observer(k) else 0)
        rc = lib().or_fcg_cb(H._h, _dptr(F), _dptr(u), rtol, maxit, C.byref(it), C.byref(rr), _dptr(hist), cb, None)
    return u, it.value, rr.value, hist[: it.value + 1], rc
