"""paper_2511_21268_b200 — B200-native solve path of arXiv 2511.21268.

fp64 PCG on the IgA Poisson stiffness system K u = F, preconditioned by one V-cycle of a
compatible-weighted-matching AMG hierarchy (Chebyshev-accelerated ℓ1-Jacobi smoothing), behind the
C ABI of ``include/amg_b200.h``.  This module is a thin binding: argument marshalling only.  PyTorch
provides device memory (caching allocator hook) and streams.

    K, F = iga_poisson(dim=3, p=3, n=96)          # generator (host, library)
    H = Hierarchy(K, params(p=3))                 # host setup + upload
    u, iters, relres, hist = H.solve(F_cuda)      # device PCG
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import AmgError, check, lib

__all__ = ["AmgError", "Hierarchy", "iga_poisson", "iga_tables", "params", "use_torch_allocator", "HostCsr",
           "Share", "setup_distributed", "set_num_threads"]


@dataclass
class HostCsr:
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray
    shape: tuple

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp
        A = sp.csr_matrix((self.data, self.indices, self.indptr), shape=self.shape)
        A.has_sorted_indices = True
        return A


def _from_c(ptr) -> HostCsr:
    rp, ci, v, shape = _lib.csr_to_numpy(ptr.contents)
    lib().amg_csr_free(ptr)
    return HostCsr(rp, ci, v, shape)


class LibCsr:
    """A library-owned amg_csr (from amg_iga_poisson with keep_c=True), for the largest workloads: no
    numpy copy of K; `Hierarchy(K, ..., take=True)` hands its arrays to amg_setup_take, after which K
    only keeps its shape.  The array views (indptr, indices, data) are valid while K is neither taken
    nor garbage-collected."""

    def __init__(self, ptr):
        self._p = ptr
        c = ptr.contents
        self.shape = (c.n_rows, c.n_cols)
        self._nnz = c.nnz

    @property
    def nnz(self) -> int:
        return self._nnz

    def _arrays(self):
        if self._p is None:
            raise ValueError("K was taken over by amg_setup_take")
        c = self._p.contents
        n, nnz = c.n_rows, c.nnz
        return (np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)),
                np.ctypeslib.as_array(c.col, shape=(max(nnz, 1),))[:nnz],
                np.ctypeslib.as_array(c.val, shape=(max(nnz, 1),))[:nnz])

    indptr = property(lambda self: self._arrays()[0])
    indices = property(lambda self: self._arrays()[1])
    data = property(lambda self: self._arrays()[2])

    def to_scipy(self):  # a copy (the views die with K)
        return HostCsr(*(a.copy() for a in self._arrays()), self.shape).to_scipy()

    def take(self):
        p, self._p = self._p, None
        if p is None:
            raise ValueError("K was already taken")
        return p

    def __del__(self):
        if getattr(self, "_p", None) is not None:
            lib().amg_csr_free(self._p)
            self._p = None


def iga_poisson(dim: int, p: int, n: int, dirichlet_sides: int = 0b000111, rhs: int = 0, geometry: int = 0,
                keep_c: bool = False):
    """amg_iga_poisson: (K as HostCsr, F as numpy fp64).  geometry 1 = the thick quarter ring (dim 3),
    geometry 2 = the three-patch L-shape (dim 3; rhs 0: f = 1, 1: F = 0, 2: its paper data).
    keep_c: K stays the library's array (LibCsr; no numpy copy) for Hierarchy(K, take=True)."""
    d = _lib.amg_iga_desc(dim, p, n, dirichlet_sides, rhs, geometry)
    Kp = C.POINTER(_lib.amg_csr)()
    Fp = C.POINTER(C.c_double)()
    check(lib().amg_iga_poisson(C.byref(d), C.byref(Kp), C.byref(Fp)))
    K = LibCsr(Kp) if keep_c else _from_c(Kp)
    F = np.ctypeslib.as_array(Fp, shape=(K.shape[0],)).copy()
    lib().amg_free(Fp)
    return K, F


def iga_tables(p: int, n: int):
    """amg_iga_tables: rounded h=1 1-D tables (M̂, K̂) in band storage (n+p, 2p+1)."""
    m = n + p
    M = np.zeros((m, 2 * p + 1))
    K = np.zeros((m, 2 * p + 1))
    dp = C.POINTER(C.c_double)
    check(lib().amg_iga_tables(p, n, M.ctypes.data_as(dp), K.ctypes.data_as(dp)))
    return M, K


def params(p: int, **overrides) -> _lib.amg_params:
    prm = _lib.amg_params()
    check(lib().amg_params_default(C.byref(prm), p))
    for k, v in overrides.items():
        if not hasattr(prm, k):
            raise AttributeError(k)
        setattr(prm, k, v)
    return prm


_ALLOC_REFS = None


def use_torch_allocator() -> None:
    """Route the library's device allocations through PyTorch's caching allocator."""
    global _ALLOC_REFS
    if _ALLOC_REFS is not None:
        return
    import torch

    ALLOC = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)
    FREE = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p)

    def _alloc(nbytes, device, stream):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device=int(device))
        except Exception:  # noqa: BLE001 — the C side reports AMG_ENOMEM
            return None

    def _free(ptr, nbytes, device, stream):
        torch.cuda.caching_allocator_delete(ptr)

    refs = (ALLOC(_alloc), FREE(_free))
    check(lib().amg_set_allocator(C.cast(refs[0], C.c_void_p), C.cast(refs[1], C.c_void_p)))
    _ALLOC_REFS = refs


def set_num_threads(n: int) -> None:
    """amg_set_num_threads: host (OpenMP) threads of this process's later library calls."""
    check(lib().amg_set_num_threads(int(n)))


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    check(lib().amg_nccl_unique_id(buf))
    return bytes(buf)


def make_dist(rank: int, nranks: int, device: int = 0, nccl_id: bytes | None = None) -> _lib.amg_dist:
    """amg_dist for one process per GPU.  Without nccl_id, rank 0 creates the NCCL unique id and it is
    broadcast with torch.distributed (the default process group must be initialised)."""
    if nccl_id is None and nranks > 1:
        import torch
        import torch.distributed as dist
        be = dist.get_backend()
        dev = torch.device("cuda", torch.cuda.current_device()) if be == "nccl" else torch.device("cpu")
        t = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nccl_id = bytes(t.cpu().numpy().tobytes())
    d = _lib.amg_dist()
    d.rank, d.nranks, d.device = rank, nranks, device
    if nccl_id is not None:
        C.memmove(d.nccl_id, nccl_id, 128)
    return d


def _borrow(K) -> tuple:
    """View a HostCsr / scipy CSR as an amg_csr (arrays kept alive by the returned tuple)."""
    indptr = np.ascontiguousarray(K.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(K.indices, dtype=np.int32)
    data = np.ascontiguousarray(K.data, dtype=np.float64)
    c = _lib.amg_csr(K.shape[0], K.shape[1], int(indptr[-1]), indptr.ctypes.data_as(C.POINTER(C.c_int64)),
                     indices.ctypes.data_as(C.POINTER(C.c_int32)), data.ctypes.data_as(C.POINTER(C.c_double)))
    return c, (indptr, indices, data)


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        return C.c_void_p(None)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


class Share:
    """amg_share_export's blob: a library-owned byte array (``array``: zero-copy uint8 view), freed
    with amg_free by ``close()`` (or garbage collection)."""

    def __init__(self, ptr: C.c_void_p, nbytes: int):
        self._p, self.nbytes = ptr, nbytes
        self.array = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(nbytes,))

    @classmethod
    def alloc(cls, nbytes: int) -> "Share":
        """A library-allocated buffer (amg_malloc) to receive a share into, for from_share(take=True)."""
        p = lib().amg_malloc(nbytes)
        if not p:
            raise MemoryError(f"amg_malloc({nbytes})")
        return cls(C.c_void_p(p), nbytes)

    def take(self) -> C.c_void_p:
        """Hand the buffer over (amg_setup_from_share_take frees it); this Share is empty afterwards."""
        p, self._p, self.array = self._p, C.c_void_p(), None
        return p

    def close(self) -> None:
        if getattr(self, "_p", None) and self._p.value:
            self.array = None
            lib().amg_free(self._p)
            self._p = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class Hierarchy:
    """amg_setup / amg_pcg_solve / amg_vcycle / amg_level_apply / export / info on one handle."""

    def __init__(self, K, prm: _lib.amg_params | None = None, dist: _lib.amg_dist | None = None,
                 take: bool = False):
        """amg_setup; take=True with a LibCsr K: amg_setup_take (K's arrays become the hierarchy's)."""
        if K is None:  # from_share
            self._h = C.c_void_p()
            return
        self._h = C.c_void_p()
        if prm is None:
            prm = params(2)
        if not prm.host_only:
            use_torch_allocator()
        dp = C.byref(dist) if dist is not None else None
        if take and isinstance(K, LibCsr):
            check(lib().amg_setup_take(K.take(), C.byref(prm), dp, C.byref(self._h)))
        else:
            c, keep = _borrow(K)
            check(lib().amg_setup(C.byref(c), C.byref(prm), dp, C.byref(self._h)))
            del keep
        self.prm = prm

    @classmethod
    def from_share(cls, share, dist: _lib.amg_dist | None = None, host_only: bool = False,
                   take: bool = False) -> "Hierarchy":
        """amg_setup_from_share: this rank's hierarchy from its blob (a Share, or any uint8 buffer).
        take=True with a Share: amg_setup_from_share_take (the blob is freed once imported)."""
        if not host_only:
            use_torch_allocator()
        H = cls(None)
        dp = C.byref(dist) if dist is not None else None
        if take and isinstance(share, Share):
            n = share.nbytes
            check(lib().amg_setup_from_share_take(share.take(), n, dp, int(host_only), C.byref(H._h)))
        else:
            arr = share.array if isinstance(share, Share) else np.ascontiguousarray(share, dtype=np.uint8)
            check(lib().amg_setup_from_share(arr.ctypes.data_as(C.c_void_p), arr.size, dp, int(host_only),
                                             C.byref(H._h)))
        H.prm = None
        return H

    def export_share(self, rank: int, nranks: int) -> Share:
        """amg_share_export: what rank `rank` of an nranks-GPU run needs from this (host) hierarchy."""
        p, n = C.c_void_p(), C.c_int64()
        check(lib().amg_share_export(self._h, rank, nranks, C.byref(p), C.byref(n)))
        return Share(p, n.value)

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            lib().amg_hierarchy_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # --- inspection ---------------------------------------------------------------------------
    def info(self) -> dict:
        nl = C.c_int64()
        N = (C.c_int64 * 32)()
        nnz = (C.c_int64 * 32)()
        nnzP = (C.c_int64 * 32)()
        opc = C.c_double()
        check(lib().amg_hierarchy_info(self._h, C.byref(nl), N, nnz, nnzP, C.byref(opc)))
        L = nl.value
        return dict(levels=L, N=list(N[:L]), nnz=list(nnz[:L]), nnz_P=list(nnzP[:L]), opc=opc.value)

    def export(self, level: int) -> dict:
        Kp, Pp = C.POINTER(_lib.amg_csr)(), C.POINTER(_lib.amg_csr)()
        ag = C.POINTER(C.c_int32)()
        dh = C.POINTER(C.c_double)()
        om = C.c_double()
        check(lib().amg_hierarchy_export(self._h, level, C.byref(Kp), C.byref(Pp), C.byref(ag), C.byref(dh),
                                         C.byref(om)))
        K = _from_c(Kp)
        n = K.shape[0]
        out = dict(K=K, P=_from_c(Pp) if Pp else None, omega=om.value)
        if ag:
            out["agg"] = np.ctypeslib.as_array(ag, shape=(n,)).copy()
            lib().amg_free(ag)
        else:
            out["agg"] = None
        out["dhat"] = np.ctypeslib.as_array(dh, shape=(n,)).copy()
        lib().amg_free(dh)
        return out

    # --- device solve path ----------------------------------------------------------------------
    def solve(self, F, u=None, rtol: float = 1e-6, maxit: int = 200, stream=None, history: bool = True):
        """amg_pcg_solve on device tensors (torch.float64, CUDA).  u: initial guess (updated in place)."""
        import torch
        if u is None:
            u = torch.zeros_like(F)
        it = C.c_int()
        rr = C.c_double()
        hist = np.full(maxit + 1, np.nan) if history else None
        st = check(lib().amg_pcg_solve(self._h, C.c_void_p(F.data_ptr()), C.c_void_p(u.data_ptr()), rtol, maxit,
                                       _stream_ptr(stream), C.byref(it), C.byref(rr),
                                       hist.ctypes.data_as(C.POINTER(C.c_double)) if history else None))
        return u, it.value, rr.value, (hist[: it.value + 1] if history else None), st

    def solve_host(self, F: np.ndarray, u: np.ndarray | None = None, rtol: float = 1e-6, maxit: int = 200,
                   stream=None):
        """amg_pcg_solve_host on host arrays (copies inside the call)."""
        F = np.ascontiguousarray(F, dtype=np.float64)
        u = np.zeros_like(F) if u is None else np.ascontiguousarray(u, dtype=np.float64)
        it = C.c_int()
        rr = C.c_double()
        dp = C.POINTER(C.c_double)
        st = check(lib().amg_pcg_solve_host(self._h, F.ctypes.data_as(dp), u.ctypes.data_as(dp), rtol, maxit,
                                            _stream_ptr(stream), C.byref(it), C.byref(rr), None))
        return u, it.value, rr.value, st

    def solve_host_ptr(self, F_ptr: int, u_ptr: int, rtol: float = 1e-6, maxit: int = 200, stream=None):
        """amg_pcg_solve_host on raw host pointers (e.g. pinned torch tensors)."""
        it = C.c_int()
        rr = C.c_double()
        dp = C.POINTER(C.c_double)
        st = check(lib().amg_pcg_solve_host(self._h, C.cast(F_ptr, dp), C.cast(u_ptr, dp), rtol, maxit,
                                            _stream_ptr(stream), C.byref(it), C.byref(rr), None))
        return it.value, rr.value, st

    def vcycle(self, r, z=None, stream=None):
        import torch
        if z is None:
            z = torch.empty_like(r)
        check(lib().amg_vcycle(self._h, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), _stream_ptr(stream)))
        return z

    def apply(self, level: int, op: int, x, y, stream=None):
        check(lib().amg_level_apply(self._h, level, op, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                    _stream_ptr(stream)))
        return y

    def set_profiling(self, enable: bool) -> None:
        check(lib().amg_set_profiling(self._h, int(enable)))

    def local_rows(self) -> tuple[int, int]:
        """This rank's rows [begin, end) of level 0 (global numbering); F and u are these rows."""
        b, e = C.c_int64(), C.c_int64()
        check(lib().amg_local_rows(self._h, C.byref(b), C.byref(e)))
        return b.value, e.value

    def dist_view(self, level: int, op: int = 0) -> dict:
        """Host view (numpy copies) of this rank's share of an operator and its halo plan."""
        v = _lib.amg_dist_view()
        check(lib().amg_dist_view_get(self._h, level, op, C.byref(v)))
        out = dict(nranks=v.nranks, replicated=bool(v.replicated))
        if v.replicated:
            return out
        nr = v.nranks
        def arr(ptr, n):
            if n <= 0 or not ptr:  # empty std::vector -> NULL data pointer
                return np.zeros(0, dtype={C.c_int64: np.int64, C.c_int32: np.int32}[ptr._type_])
            return np.ctypeslib.as_array(ptr, shape=(n,)).copy()
        rp, ci, val, shape = _lib.csr_to_numpy(v.local)
        out.update(full_cols=bool(v.full_cols), row_begin=v.row_begin, row_end=v.row_end,
                   col_begin=v.col_begin, col_end=v.col_end, ghost=arr(v.ghost, v.n_ghost), n_ghost_lo=v.n_ghost_lo,
                   send_count=arr(v.send_count, nr), send_off=arr(v.send_off, nr + 1),
                   recv_count=arr(v.recv_count, nr), recv_off=arr(v.recv_off, nr + 1),
                   local=HostCsr(rp, ci, val, shape))
        out["send_idx"] = arr(v.send_idx, int(out["send_off"][-1]))
        return out

    def op_config(self, level: int, op: int = 0) -> dict:
        c = _lib.amg_op_config()
        check(lib().amg_operator_config(self._h, level, op, C.byref(c)))
        k = c.kernel
        name = ("csr_tma" if k & 1 else "csr_regs") + ("_d16" if k & 2 else "") + \
            (f"_vi{8 * c.value_index_bytes}" if k & 8 else "") + ("_pf" if k & 4 else "")
        if c.layout == 2:
            name = "sellvi"
        if c.layout == 3:
            name = f"sellviw_b{k}"  # windows staged per CTA
        return dict(layout=("csr", "sell32", "sellvi", "sellviw")[c.layout], kernel=name, kernel_bits=k, G=c.G, U=c.U,
                    stored=c.stored, nnz=c.nnz, alg_bytes=c.alg_bytes, tuned_us=round(c.tuned_us, 2),
                    n_values=c.n_values, value_index_bytes=c.value_index_bytes, sellvi_parts=c.sellvi_parts,
                    offset_bits=c.offset_bits)

    def set_op_config(self, level: int, op: int, kernel: int, G: int, U: int) -> None:
        check(lib().amg_operator_set_config(self._h, level, op, kernel, G, U))

    def level_times(self) -> list:
        """Exclusive ms per V-cycle of every level (AMG_PROF_LEVELS=1, AMG_GRAPHS=0); resets."""
        buf = (C.c_double * 32)()
        nl = C.c_int()
        check(lib().amg_get_level_times(self._h, buf, 32, C.byref(nl)))
        return list(buf[: nl.value])

    def kernel_stats(self) -> dict:
        s = _lib.amg_kernel_stats()
        check(lib().amg_get_kernel_stats(self._h, C.byref(s)))
        return dict(launches=s.launches, total_ms=s.total_ms, bytes_per_launch=s.bytes_per_launch,
                    kernels_launched=s.kernels_launched)


def setup_distributed(K, prm: _lib.amg_params, rank: int, nranks: int, device: int = 0, group=None,
                      nccl_id: bytes | None = None, host_only: bool = False,
                      chunk_bytes: int = 1 << 28, take: bool = False) -> Hierarchy:
    """One host setup for the whole job: rank 0 builds the hierarchy of K once
    (amg_setup, host_only), exports every rank's share (amg_share_export) and sends it over `group`
    (a gloo group of torch.distributed; created when None); every rank then creates its device state
    from its own share (amg_setup_from_share).  K is only read on rank 0 (others pass None).  Plumbing
    only: the plans and the device state are the library's."""
    import torch
    import torch.distributed as dist

    import time

    ph = {}
    t0 = time.perf_counter()

    def lap(name):
        nonlocal t0
        t1 = time.perf_counter()
        ph[name] = round(ph.get(name, 0.0) + t1 - t0, 3)
        t0 = t1

    if group is None:
        group = dist.new_group(backend="gloo")
    d = make_dist(rank, nranks, device=device, nccl_id=nccl_id)
    import os
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    set_num_threads(cores)  # the host setup runs alone on rank 0: every core
    size = torch.zeros(1, dtype=torch.int64)
    lap("init")
    if rank == 0:
        hp = _lib.amg_params()
        C.memmove(C.byref(hp), C.byref(prm), C.sizeof(hp))
        hp.host_only = 1
        G = Hierarchy(K, hp, take=take)  # take: K's arrays become G's level 0 (one copy of K₀ less)
        lap("host_setup")
        # the other ranks' shares first, one at a time; rank 0's own last, after which the global
        # hierarchy is freed before rank 0's device setup (host RAM holds at most G + one share + the
        # receiving rank's upload at any time)
        for q in list(range(1, nranks)) + [0]:
            sh = G.export_share(q, nranks)
            lap("export")
            ph["share_bytes"] = ph.get("share_bytes", 0) + sh.nbytes
            if q == 0:
                mine = sh
                continue
            size[0] = sh.nbytes
            dist.send(size, q, group=group)
            t = torch.from_numpy(sh.array)
            for o in range(0, sh.nbytes, chunk_bytes):
                dist.send(t[o:o + chunk_bytes], q, group=group)
            sh.close()
            lap("send")
        G.close()
        set_num_threads(max(1, cores // nranks))  # the device setups run side by side
        H = Hierarchy.from_share(mine, d, host_only=host_only, take=True)
    else:
        dist.recv(size, 0, group=group)
        lap("wait")
        sh = Share.alloc(int(size[0]))  # the library frees it once imported (from_share take=True)
        buf = torch.from_numpy(sh.array)
        for o in range(0, buf.numel(), chunk_bytes):
            dist.recv(buf[o:o + chunk_bytes], 0, group=group)
        del buf
        lap("recv")
        set_num_threads(max(1, cores // nranks))
        H = Hierarchy.from_share(sh, d, host_only=host_only, take=True)
    lap("device_setup")
    H.prm = prm
    H.setup_phases = ph
    return H
