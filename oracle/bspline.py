"""Floating-point B-spline evaluation, Gauss quadrature, element-loop assembly, load vector and
L2 error (oracle; c.1, c.2, c.4 cross-check, c.5 of SURVEY.md §8c).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

Paper passages:
  * basis / open knot vectors / C^{p-1}: P:L69-78, P:L1105, P:L1124;
  * single-patch Galerkin assembly with (p+1)^d Gauss points per element: P:L551-568, Remark P:L570-573;
  * Dirichlet DOFs fixed (eliminated): P:L566-567, cube sides P:L1061-1072 (Dirichlet on 3 faces).

Numbering (c.1): functions a = 0..m-1 per axis (m = n+p); free DOFs are numbered lexicographically
with x fastest over the free index ranges.  Sides: 1:x=0 2:x=1 3:y=0 4:y=1 5:z=0 6:z=1.
"""
from __future__ import annotations

import numpy as np


def knots(p: int, n: int) -> np.ndarray:
    """Open uniform knot vector on [0,1] with n elements."""
    return np.concatenate([np.zeros(p), np.linspace(0.0, 1.0, n + 1), np.ones(p)])


def eval_basis(p: int, n: int, x: np.ndarray, deriv: bool = False) -> np.ndarray:
    """All m=n+p basis functions (or derivatives) at points x: Cox–de Boor recursion.

    Returns an array (len(x), m).  x=1 is assigned to the last element.
    """
    t = knots(p, n)
    m = n + p
    x = np.asarray(x, dtype=np.float64)
    # degree-0
    N = np.zeros((x.size, len(t) - 1))
    span = np.minimum(np.floor(x * n).astype(int), n - 1) + p
    N[np.arange(x.size), span] = 1.0
    dN = None
    for k in range(1, p + 1):
        Nn = np.zeros((x.size, len(t) - 1 - k))
        for i in range(len(t) - 1 - k):
            d1 = t[i + k] - t[i]
            d2 = t[i + k + 1] - t[i + 1]
            if d1 > 0:
                Nn[:, i] += (x - t[i]) / d1 * N[:, i]
            if d2 > 0:
                Nn[:, i] += (t[i + k + 1] - x) / d2 * N[:, i + 1]
        if k == p and deriv:
            # N'_{i,p} = p/(t_{i+p}-t_i) N_{i,p-1} - p/(t_{i+p+1}-t_{i+1}) N_{i+1,p-1}
            dN = np.zeros((x.size, m))
            for i in range(m):
                d1 = t[i + p] - t[i]
                d2 = t[i + p + 1] - t[i + 1]
                if d1 > 0:
                    dN[:, i] += p / d1 * N[:, i]
                if d2 > 0:
                    dN[:, i] -= p / d2 * N[:, i + 1]
        N = Nn
    return dN if deriv else N[:, :m]


def gauss(npts: int):
    """Gauss–Legendre rule on [0,1]."""
    xg, wg = np.polynomial.legendre.leggauss(npts)
    return 0.5 * (xg + 1.0), 0.5 * wg


def free_range(m: int, ax: int, dirichlet_sides: int):
    lo = 1 if dirichlet_sides >> (2 * ax) & 1 else 0
    hi = m - 1 - (1 if dirichlet_sides >> (2 * ax + 1) & 1 else 0)
    return lo, hi


def element_loop_matrices_1d(p: int, n: int):
    """1-D mass and stiffness by an element loop with (p+1) Gauss points (dense m×m, fp64)."""
    m = n + p
    xg, wg = gauss(p + 1)
    M = np.zeros((m, m))
    K = np.zeros((m, m))
    for e in range(n):
        x = (e + xg) / n
        w = wg / n
        B = eval_basis(p, n, x)
        dB = eval_basis(p, n, x, deriv=True)
        M += (B * w[:, None]).T @ B
        K += (dB * w[:, None]).T @ dB
    return M, K


def element_loop_stiffness(dim: int, p: int, n: int, dirichlet_sides: int = 0b000111) -> np.ndarray:
    """Dense d-dimensional stiffness k_ij = ∫∇φ_j·∇φ_i by a genuine d-D element loop with (p+1)^d
    Gauss points, J_F = I on the unit square/cube, then Dirichlet elimination.

    Independent of the Kronecker-sum route used by oracle.c; only for small n (dense output).
    """
    m = n + p
    xg, wg = gauss(p + 1)
    ndof = m ** dim
    K = np.zeros((ndof, ndof))
    for elem in np.ndindex(*([n] * dim)):
        # quadrature points of this element
        pts_1d = [(elem[ax] + xg) / n for ax in range(dim)]
        B = [eval_basis(p, n, pts_1d[ax]) for ax in range(dim)]
        dB = [eval_basis(p, n, pts_1d[ax], deriv=True) for ax in range(dim)]
        act = [np.arange(elem[ax], elem[ax] + p + 1) for ax in range(dim)]
        for q in np.ndindex(*([p + 1] * dim)):
            wq = np.prod([wg[q[ax]] / n for ax in range(dim)])
            vals = []
            grads = []
            idx = []
            for loc in np.ndindex(*([p + 1] * dim)):
                fn = [act[ax][loc[ax]] for ax in range(dim)]
                v = np.prod([B[ax][q[ax], fn[ax]] for ax in range(dim)])
                g = []
                for dax in range(dim):
                    g.append(np.prod([(dB if ax == dax else B)[ax][q[ax], fn[ax]] for ax in range(dim)]))
                gi = 0
                for ax in reversed(range(dim)):
                    gi = gi * m + fn[ax]
                idx.append(gi)
                vals.append(v)
                grads.append(g)
            G = np.array(grads)
            K[np.ix_(idx, idx)] += wq * (G @ G.T)
    keep = free_index_list(dim, m, dirichlet_sides)
    return K[np.ix_(keep, keep)]


def free_index_list(dim: int, m: int, dirichlet_sides: int) -> np.ndarray:
    """Global (all-DOF, x-fastest) indices of the free DOFs in free-lexicographic order (c.1/c.2)."""
    ranges = [free_range(m, ax, dirichlet_sides) for ax in range(dim)]
    grids = [np.arange(lo, hi + 1) for lo, hi in ranges]
    if dim == 2:
        yy, xx = np.meshgrid(grids[1], grids[0], indexing="ij")
        return (xx + m * yy).ravel()
    zz, yy, xx = np.meshgrid(grids[2], grids[1], grids[0], indexing="ij")
    return (xx + m * (yy + m * zz)).ravel()


# --- manufactured solution (c.5): u* = sin(πx) sin(πy/2) [cos(πz)] ------------------------------
_FACT = [lambda x: np.sin(np.pi * x), lambda y: np.sin(0.5 * np.pi * y), lambda z: np.cos(np.pi * z)]


def manufactured_u(dim: int, *xyz):
    u = 1.0
    for ax in range(dim):
        u = u * _FACT[ax](xyz[ax])
    return u


def source_factor(dim: int) -> float:
    """−Δu* = c·u*: c = π²(1 + 1/4) in 2-D, π²(1 + 1/4 + 1) = 9π²/4 in 3-D."""
    return (5.0 if dim == 2 else 9.0) * np.pi ** 2 / 4.0


def load_vector(dim: int, p: int, n: int, dirichlet_sides: int = 0b000111) -> np.ndarray:
    """F_i = ∫ f φ_i (eq:matrix_and_vector_values P:L646-650) for f = c·u*, which is separable:
    F = c · F_x ⊗ F_y (⊗ F_z), each 1-D factor by (p+1)-point Gauss per element.
    u* vanishes on sides 1-3 and has zero normal derivative on sides 4-6, so no lifting and no
    Neumann integral is needed (SURVEY c.5)."""
    m = n + p
    xg, wg = gauss(p + 1)
    f1 = []
    for ax in range(dim):
        F = np.zeros(m)
        for e in range(n):
            x = (e + xg) / n
            B = eval_basis(p, n, x)
            F += (B * (wg / n * _FACT[ax](x))[:, None]).sum(axis=0)
        lo, hi = free_range(m, ax, dirichlet_sides)
        f1.append(F[lo:hi + 1])
    out = f1[0]
    for ax in range(1, dim):
        out = np.kron(f1[ax], out)  # x fastest
    return source_factor(dim) * out


def l2_error(dim: int, p: int, n: int, u_free: np.ndarray, dirichlet_sides: int = 0b000111) -> float:
    """‖u_h − u*‖_{L2(Ω)} by (p+2)^d Gauss points per element (u_h = 0 on eliminated DOFs)."""
    m = n + p
    coef = np.zeros(m ** dim)
    coef[free_index_list(dim, m, dirichlet_sides)] = u_free
    coef = coef.reshape([m] * dim)  # x fastest -> array index order (z,) y, x
    xg, wg = gauss(p + 2)
    pts = np.concatenate([(e + xg) / n for e in range(n)])
    wts = np.concatenate([wg / n for _ in range(n)])
    B = eval_basis(p, n, pts)  # (Q, m)
    if dim == 2:
        uh = np.einsum("qx,yx,ry->rq", B, coef, B)  # r: y point, q: x point
        X, Y = pts[None, :], pts[:, None]
        err = (uh - manufactured_u(2, X, Y)) ** 2
        return float(np.sqrt(np.einsum("r,q,rq->", wts, wts, err)))
    uh = np.einsum("ax,zyx->zya", B, coef)
    uh = np.einsum("by,zya->zba", B, uh)
    uh = np.einsum("cz,zba->cba", B, uh)  # (z_q, y_q, x_q)
    Z, Y, X = np.meshgrid(pts, pts, pts, indexing="ij")
    err = (uh - manufactured_u(3, X, Y, Z)) ** 2
    return float(np.sqrt(np.einsum("c,b,a,cba->", wts, wts, wts, err)))
