"""The paper's cube experiment with its own data: load vector with inhomogeneous
Dirichlet data (L2 boundary projection + lifting) and Neumann face integrals, and the L2 error of the
discrete solution including its Dirichlet part.

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

Problem ("Cube"): −Δu = f on Ω = [0,1]³ with
    f = −e^{x+z} sin y,   g_D = e^{x+z} sin y on sides 1, 2, 3 (x=0, x=1, y=0),
    g_N = e^{x+z} cos y (side 4, y=1),  −e^{x+z} sin y (side 5, z=0),  e^{x+z} sin y (side 6, z=1),
whose exact solution is u = e^{x+z} sin y.  Discretisation (eq:matrix_and_vector_values
P:L646-650): Galerkin with the tensor B-spline space of degree p, C^{p−1}, on n³ elements; integrals by
(p+1)-point Gauss per element and direction (Remark P:L570-573).

Readings (NEXT-1):
  * Dirichlet data: GeoPDEs-style L2 projection of g_D onto the trace space of the union of the
    Dirichlet faces — ONE boundary mass system over all Dirichlet DOFs, each face contributing its 2-D
    mass matrix and load (DOFs on an edge shared by two Dirichlet faces receive both contributions).
  * The free-DOF system is K_ff u_f = F_f − K_fD u_D, with F the source + Neumann load of the free DOFs.

Numbering: functions a = 0..m−1 per axis (m = n+p), all-DOF index a + m(b + m c) (x fastest); the free
DOFs are the free-lexicographic subset (bspline.free_index_list).

Two independent routes:
  * ``paper_cube_rhs``  — the separable fast path (1-D factors, tensor contractions), any n;
  * ``generic_rhs``     — plain element / face loops with callables f, g_D, g_N, small n; it is also
                           how the polynomial-reproduction pin is computed.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .bspline import element_loop_matrices_1d, eval_basis, free_index_list, free_range, gauss

DIRICHLET = (1, 2, 3)  # sides with Dirichlet data
NEUMANN = (4, 5, 6)


def _side_axis(side: int):
    """side s (1..6) -> (axis, end) with end 0 (coordinate 0) or 1 (coordinate 1)."""
    return (side - 1) // 2, (side - 1) % 2


def _quad_1d(p: int, n: int):
    """All (p+1)-point Gauss nodes / weights of the n elements of [0,1] and the basis values there."""
    xg, wg = gauss(p + 1)
    x = np.concatenate([(e + xg) / n for e in range(n)])
    w = np.concatenate([wg / n for _ in range(n)])
    return x, w, eval_basis(p, n, x)


# ------------------------------------------------------------------------------------------------
# generic route: callables, element loops (small n)
# ------------------------------------------------------------------------------------------------
def generic_rhs(p: int, n: int, f, gD, gN: dict):
    """(F_free, u_D_all) for −Δu = f with g_D on DIRICHLET sides and g_N[side] on NEUMANN sides, by
    plain quadrature over the volume / faces ((p+1)^d Gauss points per element)."""
    m = n + p
    x, w, B = _quad_1d(p, n)
    # volume load: F[a,b,c] = Σ_q f(x_q) N_a N_b N_c w  (array index order c, b, a)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")  # (x, y, z) point grids, index order (ix, iy, iz)
    fv = f(X, Y, Z) * (w[:, None, None] * w[None, :, None] * w[None, None, :])
    Fall = np.einsum("ijk,ia,jb,kc->cba", fv, B, B, B)
    # Neumann faces
    for side, g in gN.items():
        ax, end = _side_axis(side)
        coord = float(end)
        N1 = eval_basis(p, n, np.array([coord]))[0]  # basis values on the face coordinate
        U, V = np.meshgrid(x, x, indexing="ij")
        ww = w[:, None] * w[None, :]
        if ax == 0:
            gv = g(np.full_like(U, coord), U, V) * ww  # (y, z)
            Fall += np.einsum("jk,jb,kc,a->cba", gv, B, B, N1)
        elif ax == 1:
            gv = g(U, np.full_like(U, coord), V) * ww  # (x, z)
            Fall += np.einsum("ik,ia,kc,b->cba", gv, B, B, N1)
        else:
            gv = g(U, V, np.full_like(U, coord)) * ww  # (x, y)
            Fall += np.einsum("ij,ia,jb,c->cba", gv, B, B, N1)
    uD = dirichlet_projection_generic(p, n, gD)
    return _lift(p, n, Fall.ravel(), uD), uD


def dirichlet_projection_generic(p: int, n: int, gD) -> np.ndarray:
    """All-DOF vector holding the joint L2 projection of g_D on the Dirichlet faces (0 elsewhere)."""
    m = n + p
    x, w, B = _quad_1d(p, n)
    Mx, _ = element_loop_matrices_1d(p, n)
    dofs = _dirichlet_dofs(m)
    pos = {int(g): k for k, g in enumerate(dofs)}
    nd = len(dofs)
    Mb = np.zeros((nd, nd))
    rhs = np.zeros(nd)
    for side in DIRICHLET:
        ax, end = _side_axis(side)
        idx_fixed = 0 if end == 0 else m - 1
        coord = float(end)
        U, V = np.meshgrid(x, x, indexing="ij")
        ww = w[:, None] * w[None, :]
        # the two in-face axes (ascending) and the face DOFs
        fa = [a for a in range(3) if a != ax]
        pts = [None, None, None]
        pts[ax] = np.full_like(U, coord)
        pts[fa[0]] = U
        pts[fa[1]] = V
        gv = gD(*pts) * ww
        Fface = np.einsum("uv,ua,vb->ab", gv, B, B)  # (first in-face axis, second)
        for i0 in range(m):
            for i1 in range(m):
                ind = [0, 0, 0]
                ind[ax] = idx_fixed
                ind[fa[0]] = i0
                ind[fa[1]] = i1
                gi = ind[0] + m * (ind[1] + m * ind[2])
                rhs[pos[gi]] += Fface[i0, i1]
                for j0 in range(max(0, i0 - p), min(m, i0 + p + 1)):
                    for j1 in range(max(0, i1 - p), min(m, i1 + p + 1)):
                        jnd = [0, 0, 0]
                        jnd[ax] = idx_fixed
                        jnd[fa[0]] = j0
                        jnd[fa[1]] = j1
                        gj = jnd[0] + m * (jnd[1] + m * jnd[2])
                        Mb[pos[gi], pos[gj]] += Mx[i0, j0] * Mx[i1, j1]
    uD = np.zeros(m ** 3)
    uD[dofs] = np.linalg.solve(Mb, rhs)
    return uD


def _dirichlet_dofs(m: int) -> np.ndarray:
    """All-DOF indices on the Dirichlet faces (sides 1, 2, 3), ascending."""
    a, b, c = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    on = (a == 0) | (a == m - 1) | (b == 0)
    return np.sort((a + m * (b + m * c))[on])


def _lift(p: int, n: int, Fall: np.ndarray, uD: np.ndarray) -> np.ndarray:
    """F_free = F_all[free] − (K_full u_D)[free], K_full = K⊗M⊗M + M⊗K⊗M + M⊗M⊗K (all DOFs)."""
    m = n + p
    M1, K1 = element_loop_matrices_1d(p, n)
    U = uD.reshape(m, m, m)  # (c, b, a)

    def apply(Az, Ay, Ax):
        t = np.einsum("ad,cbd->cba", Ax, U)
        t = np.einsum("bd,cda->cba", Ay, t)
        return np.einsum("cd,dba->cba", Az, t)

    KU = apply(M1, M1, K1) + apply(M1, K1, M1) + apply(K1, M1, M1)
    free = free_index_list(3, m, 0b000111)
    return (Fall - KU.ravel())[free]


# ------------------------------------------------------------------------------------------------
# the paper's data, separable route (any n)
# ------------------------------------------------------------------------------------------------
def _moments(p: int, n: int, fn) -> np.ndarray:
    """∫_0^1 fn(t) N_a(t) dt for all a, (p+1)-point Gauss per element."""
    x, w, B = _quad_1d(p, n)
    return (B * (w * fn(x))[:, None]).sum(axis=0)


def paper_cube_rhs(p: int, n: int):
    """(F_free, u_D_all) of the paper's cube by the separable route:
      source  −e^x·sin y·e^z          → −(E_x ⊗ S_y ⊗ E_z)
      side 4  e^x·cos(1)·e^z, b = m−1  → cos 1 · E_x ⊗ e_{m−1} ⊗ E_z
      side 5  −e^x·sin y, c = 0        → −E_x ⊗ S_y ⊗ e_0
      side 6  e·e^x·sin y, c = m−1      → e · E_x ⊗ S_y ⊗ e_{m−1}
    (N_b(1) = δ_{b,m−1}, N_c(0) = δ_{c,0} on open knot vectors), then the joint boundary projection of
    g_D (faces x=0: e^z sin y, x=1: e·e^z sin y, y=0: 0) and the lifting."""
    m = n + p
    E = _moments(p, n, np.exp)
    S = _moments(p, n, np.sin)
    Fall = -np.einsum("c,b,a->cba", E, S, E)
    e_last = np.zeros(m)
    e_last[-1] = 1.0
    e_first = np.zeros(m)
    e_first[0] = 1.0
    Fall += np.cos(1.0) * np.einsum("c,b,a->cba", E, e_last, E)
    Fall += -np.einsum("c,b,a->cba", e_first, S, E)
    Fall += np.e * np.einsum("c,b,a->cba", e_last, S, E)
    uD = dirichlet_projection_sparse(p, n)
    return _lift(p, n, Fall.ravel(), uD), uD


def dirichlet_projection_sparse(p: int, n: int) -> np.ndarray:
    """Joint L2 projection of the paper's g_D on the Dirichlet faces as a sparse boundary mass system
    (same system as dirichlet_projection_generic; face mass = M ⊗ M of the two in-face directions,
    face load = separable moments)."""
    m = n + p
    M1, _ = element_loop_matrices_1d(p, n)
    E = _moments(p, n, np.exp)
    S = _moments(p, n, np.sin)
    dofs = _dirichlet_dofs(m)
    pos = -np.ones(m ** 3, dtype=np.int64)
    pos[dofs] = np.arange(len(dofs))
    Mc = sp.csr_matrix(M1)
    rows, cols, vals = [], [], []
    rhs = np.zeros(len(dofs))
    i0, i1 = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    FM = sp.kron(Mc, Mc).tocoo()  # (i0*m + i1, j0*m + j1) pairs with M[i0,j0]*M[i1,j1]
    for side in DIRICHLET:
        ax, end = _side_axis(side)
        fixed = 0 if end == 0 else m - 1

        def gidx(u, v):
            ind = [None, None, None]
            fa = [a for a in range(3) if a != ax]
            ind[ax] = fixed
            ind[fa[0]] = u
            ind[fa[1]] = v
            return ind[0] + m * (ind[1] + m * ind[2])

        r = pos[gidx(FM.row // m, FM.row % m)]
        c = pos[gidx(FM.col // m, FM.col % m)]
        rows.append(r)
        cols.append(c)
        vals.append(FM.data)
        # face load of g_D: x=0 → e^z sin y (in-face axes y, z), x=1 → e·e^z sin y, y=0 → 0
        if side in (1, 2):
            scale = 1.0 if side == 1 else np.e
            Fface = scale * np.einsum("u,v->uv", S, E)  # (y, z)
            rhs[pos[gidx(i0, i1)]] += Fface
    Mb = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                       shape=(len(dofs), len(dofs)))
    uD = np.zeros(m ** 3)
    uD[dofs] = spla.spsolve(Mb.tocsc(), rhs)
    return uD


def exact_u(x, y, z):
    return np.exp(x + z) * np.sin(y)


def l2_error_full(p: int, n: int, u_free: np.ndarray, uD: np.ndarray, exact=exact_u) -> float:
    """‖u_h − u‖_{L2(Ω)} with u_h = free part + Dirichlet part, (p+2)³ Gauss points per element."""
    m = n + p
    coef = uD.copy()
    coef[free_index_list(3, m, 0b000111)] = u_free
    coef = coef.reshape(m, m, m)  # (c, b, a)
    xg, wg = gauss(p + 2)
    pts = np.concatenate([(e + xg) / n for e in range(n)])
    wts = np.concatenate([wg / n for _ in range(n)])
    B = eval_basis(p, n, pts)
    uh = np.einsum("ax,zyx->zya", B, coef)
    uh = np.einsum("by,zya->zba", B, uh)
    uh = np.einsum("cz,zba->cba", B, uh)  # (z_q, y_q, x_q)
    Zq, Yq, Xq = np.meshgrid(pts, pts, pts, indexing="ij")
    err = (uh - exact(Xq, Yq, Zq)) ** 2
    return float(np.sqrt(np.einsum("c,b,a,cba->", wts, wts, wts, err)))


def paper_cube_generic(p: int, n: int):
    """The paper's data through the generic route (pins the separable route)."""
    f = lambda x, y, z: -np.exp(x + z) * np.sin(y)  # noqa: E731
    gD = exact_u
    gN = {4: lambda x, y, z: np.exp(x + z) * np.cos(y),
          5: lambda x, y, z: -np.exp(x + z) * np.sin(y),
          6: lambda x, y, z: np.exp(x + z) * np.sin(y)}
    return generic_rhs(p, n, f, gD, gN)
