"""The thick quarter ring (§3.3): a
non-isoparametric discretisation — NURBS geometry, B-spline solution space — of −Δu = f.

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

Geometry (inner radius 1, outer radius 2, height 1, in the positive orthant).  Reading
(R.a): the GeoPDEs-style parametrisation
    x = r(u)·c_x(v),  y = r(u)·c_y(v),  z = w,   r(u) = 1 + u,
with c(v) the rational quadratic quarter circle (control points (1,0), (1,1), (0,1), weights
(1, √2/2, 1)) — the exact NURBS circle; sides 1: u=0 (r=1), 2: u=1 (r=2), 3: v=0 (y=0 plane),
4: v=1 (x=0 plane), 5: w=0, 6: w=1; Dirichlet on sides 1-3, Neumann on 4-6.

Stiffness (non-isoparametric entries k_ij = ∫ ∇_ξN_jᵀ J⁻¹J⁻ᵀ ∇_ξN_i det J dξ).  Because
|c| = 1 and c·c' = 0, JᵀJ = diag(1, r²|c'|², 1) and det J = r|c'|, so the integrand separates:
    K = A_u ⊗ B_v ⊗ M_w + C_u ⊗ D_v ⊗ M_w + E_u ⊗ B_v ⊗ K_w        (x fastest = u, then v, then w)
    A_u = ∫ N'N' r du,  C_u = ∫ N N /r du,  E_u = ∫ N N r du,
    B_v = ∫ N N |c'| dv, D_v = ∫ N'N' /|c'| dv,  M_w = ∫ N N dw,  K_w = ∫ N'N' dw,
each integral by (p+1)-point Gauss per element (the paper's quadrature; not exact for the
rational weights).  The 1-D tables are evaluated in 50-digit decimal arithmetic and rounded once to
fp64 (correctly rounded), then every 3-D entry is ((A·B)·M + (C·D)·M) + (E·B)·K in that order — the
canonical contract of DESIGN.md §3, so an independent implementation can match it bitwise.
"""
from __future__ import annotations

import decimal
from decimal import Decimal as D

import numpy as np
import scipy.sparse as sp

from .bspline import eval_basis, free_index_list, gauss

_CTX = decimal.Context(prec=50)


# ------------------------------------------------------------------------------------------------
# high-precision 1-D quadrature
# ------------------------------------------------------------------------------------------------
def _gauss_dec(npts: int):
    """Gauss–Legendre nodes/weights on [0,1], 50 digits (Newton on P_n from the fp64 roots)."""
    with decimal.localcontext(_CTX):
        xs, ws = [], []
        x0, _ = np.polynomial.legendre.leggauss(npts)
        for z0 in x0:
            z = D(repr(float(z0)))
            for _ in range(60):
                p0, p1 = D(1), z
                for k in range(2, npts + 1):
                    p0, p1 = p1, ((2 * k - 1) * z * p1 - (k - 1) * p0) / k
                if npts == 1:
                    p0, p1 = D(1), z
                dp = npts * (z * p1 - p0) / (z * z - 1)
                dz = p1 / dp
                z -= dz
                if abs(dz) < D("1e-48"):
                    break
            p0, p1 = D(1), z
            for k in range(2, npts + 1):
                p0, p1 = p1, ((2 * k - 1) * z * p1 - (k - 1) * p0) / k
            if npts == 1:
                p0, p1 = D(1), z
            dp = npts * (z * p1 - p0) / (z * z - 1)
            xs.append((z + 1) / 2)
            ws.append(1 / ((1 - z * z) * dp * dp))
        return xs, ws


def _basis_dec(p: int, n: int, x: D):
    """All m = n+p B-spline values and derivatives at x ∈ [0,1] (open uniform knots i/n), decimal."""
    with decimal.localcontext(_CTX):
        m = n + p
        t = [D(0)] * p + [D(i) / n for i in range(n + 1)] + [D(1)] * p
        span = min(int(x * n), n - 1) + p
        N = [D(0)] * (len(t) - 1)
        N[span] = D(1)
        dN = None
        for k in range(1, p + 1):
            Nn = [D(0)] * (len(t) - 1 - k)
            for i in range(len(t) - 1 - k):
                d1 = t[i + k] - t[i]
                d2 = t[i + k + 1] - t[i + 1]
                v = D(0)
                if d1 > 0:
                    v += (x - t[i]) / d1 * N[i]
                if d2 > 0:
                    v += (t[i + k + 1] - x) / d2 * N[i + 1]
                Nn[i] = v
            if k == p:
                dN = [D(0)] * m
                for i in range(m):
                    d1 = t[i + p] - t[i]
                    d2 = t[i + p + 1] - t[i + 1]
                    if d1 > 0:
                        dN[i] += p / d1 * N[i]
                    if d2 > 0:
                        dN[i] -= p / d2 * N[i + 1]
            N = Nn
        return N[:m], dN


def _circle_speed(v: D) -> D:
    """|c'(v)| of the rational quadratic quarter circle (weights 1, √2/2, 1)."""
    with decimal.localcontext(_CTX):
        w1 = D(2).sqrt() / 2
        one = D(1)
        X = (one - v) ** 2 + 2 * v * (one - v) * w1
        Y = 2 * v * (one - v) * w1 + v * v
        W = (one - v) ** 2 + 2 * v * (one - v) * w1 + v * v
        Xp = -2 * (one - v) + 2 * w1 * (one - 2 * v)
        Yp = 2 * w1 * (one - 2 * v) + 2 * v
        Wp = -2 * (one - v) + 2 * w1 * (one - 2 * v) + 2 * v
        cx = (Xp * W - X * Wp) / (W * W)
        cy = (Yp * W - Y * Wp) / (W * W)
        return (cx * cx + cy * cy).sqrt()


def weighted_tables(p: int, n: int):
    """Correctly-rounded fp64 1-D tables (dense m×m): A_u, C_u, E_u, B_v, D_v, M_w, K_w."""
    m = n + p
    xg, wg = _gauss_dec(p + 1)
    acc = {k: [[D(0)] * m for _ in range(m)] for k in ("A", "C", "E", "B", "Dv", "M", "K")}
    with decimal.localcontext(_CTX):
        h = D(1) / n
        for e in range(n):
            for q in range(p + 1):
                x = (e + xg[q]) * h
                w = wg[q] * h
                N, dN = _basis_dec(p, n, x)
                r = 1 + x
                s = _circle_speed(x)
                for i in range(e, e + p + 1):
                    for j in range(e, e + p + 1):
                        nn, dd = N[i] * N[j] * w, dN[i] * dN[j] * w
                        acc["A"][i][j] += dd * r
                        acc["C"][i][j] += nn / r
                        acc["E"][i][j] += nn * r
                        acc["B"][i][j] += nn * s
                        acc["Dv"][i][j] += dd / s
                        acc["M"][i][j] += nn
                        acc["K"][i][j] += dd
    return {k: np.array([[float(v) for v in row] for row in T]) for k, T in acc.items()}


# ------------------------------------------------------------------------------------------------
# stiffness (canonical Kronecker route) and an independent 3-D element loop
# ------------------------------------------------------------------------------------------------
def assemble_ring(p: int, n: int, tables=None, dirichlet_sides: int = 0b000111) -> sp.csr_matrix:
    """Free-DOF stiffness of the quarter ring, structural (2p+1)³ pattern, canonical op order."""
    T = tables or weighted_tables(p, n)
    m = n + p
    free = free_index_list(3, m, dirichlet_sides)
    pos = -np.ones(m ** 3, dtype=np.int64)
    pos[free] = np.arange(len(free))
    rows, cols, vals = [], [], []
    offs = np.arange(-p, p + 1)
    for gi, g in enumerate(free):
        a, b, c = g % m, (g // m) % m, g // (m * m)
        c2 = c + offs
        b2 = b + offs
        a2 = a + offs
        c2 = c2[(c2 >= 0) & (c2 < m)]
        b2 = b2[(b2 >= 0) & (b2 < m)]
        a2 = a2[(a2 >= 0) & (a2 < m)]
        C2, B2, A2 = np.meshgrid(c2, b2, a2, indexing="ij")
        gj = (A2 + m * (B2 + m * C2)).ravel()
        keep = pos[gj] >= 0
        A2, B2, C2 = A2.ravel()[keep], B2.ravel()[keep], C2.ravel()[keep]
        t1 = (T["A"][a, A2] * T["B"][b, B2]) * T["M"][c, C2]
        t2 = (T["C"][a, A2] * T["Dv"][b, B2]) * T["M"][c, C2]
        t3 = (T["E"][a, A2] * T["B"][b, B2]) * T["K"][c, C2]
        rows.append(np.full(keep.sum(), gi))
        cols.append(pos[gj[keep]])
        vals.append((t1 + t2) + t3)
    N = len(free)
    K = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
    K.sort_indices()
    return K


def geometry(u, v, w):
    """Physical point and the Jacobian pieces (r, c, c') at parametric (u, v, w), fp64."""
    w1 = np.sqrt(2.0) / 2.0
    X = (1 - v) ** 2 + 2 * v * (1 - v) * w1
    Y = 2 * v * (1 - v) * w1 + v * v
    W = (1 - v) ** 2 + 2 * v * (1 - v) * w1 + v * v
    Xp = -2 * (1 - v) + 2 * w1 * (1 - 2 * v)
    Yp = 2 * w1 * (1 - 2 * v) + 2 * v
    Wp = -2 * (1 - v) + 2 * w1 * (1 - 2 * v) + 2 * v
    cx, cy = X / W, Y / W
    dcx, dcy = (Xp * W - X * Wp) / W ** 2, (Yp * W - Y * Wp) / W ** 2
    r = 1 + u
    return r * cx, r * cy, w, (r, cx, cy, dcx, dcy)


def element_loop_ring(p: int, n: int) -> np.ndarray:
    """Dense free-DOF stiffness by a genuine 3-D element loop with the full Jacobian J⁻¹J⁻ᵀ det J at
    (p+1)³ Gauss points (fp64): the non-isoparametric formula P:L598-603 applied directly (small n)."""
    m = n + p
    xg, wg = gauss(p + 1)
    Kd = np.zeros((m ** 3, m ** 3))
    for e in np.ndindex(n, n, n):
        pts = [(e[ax] + xg) / n for ax in range(3)]
        B = [eval_basis(p, n, pts[ax]) for ax in range(3)]
        dB = [eval_basis(p, n, pts[ax], deriv=True) for ax in range(3)]
        act = [np.arange(e[ax], e[ax] + p + 1) for ax in range(3)]
        for q in np.ndindex(p + 1, p + 1, p + 1):
            u, v, w = pts[0][q[0]], pts[1][q[1]], pts[2][q[2]]
            _, _, _, (r, cx, cy, dcx, dcy) = geometry(u, v, w)
            J = np.array([[cx, r * dcx, 0.0], [cy, r * dcy, 0.0], [0.0, 0.0, 1.0]])
            Ji = np.linalg.inv(J)
            G = Ji @ Ji.T * abs(np.linalg.det(J))
            wq = wg[q[0]] * wg[q[1]] * wg[q[2]] / n ** 3
            idx, grads = [], []
            for loc in np.ndindex(p + 1, p + 1, p + 1):
                fa, fb, fc = act[0][loc[0]], act[1][loc[1]], act[2][loc[2]]
                gx = dB[0][q[0], fa] * B[1][q[1], fb] * B[2][q[2], fc]
                gy = B[0][q[0], fa] * dB[1][q[1], fb] * B[2][q[2], fc]
                gz = B[0][q[0], fa] * B[1][q[1], fb] * dB[2][q[2], fc]
                idx.append(fa + m * (fb + m * fc))
                grads.append((gx, gy, gz))
            Gr = np.array(grads)
            Kd[np.ix_(idx, idx)] += wq * (Gr @ G @ Gr.T)
    keep = free_index_list(3, m, 0b000111)
    return Kd[np.ix_(keep, keep)]


# ------------------------------------------------------------------------------------------------
# the paper's ring data (P:L1093-1102 with eq:Lshapedcoeff P:L1079-1089): plain quadrature, small n
# ------------------------------------------------------------------------------------------------
def exact_u(x, y, z):
    return np.exp(x) * np.sin(x * y) * np.cos(z)


def _f(x, y, z):
    return np.exp(x) * np.cos(z) * (-2.0 * np.cos(x * y) * y + np.sin(x * y) * (y * y + x * x))


_GN = {4: lambda x, y, z: -np.exp(x) * np.cos(z) * (np.sin(x * y) + y * np.cos(x * y)),
       5: lambda x, y, z: np.exp(x) * np.sin(x * y) * np.sin(z),
       6: lambda x, y, z: -np.exp(x) * np.sin(x * y) * np.sin(z)}


def _speed(v):
    _, _, _, (r, cx, cy, dcx, dcy) = geometry(np.zeros_like(v), v, np.zeros_like(v))
    return np.sqrt(dcx * dcx + dcy * dcy)


def paper_ring_rhs(p: int, n: int):
    """(F_free, u_D_all) of the paper's ring problem: source ∫ f N det J, Neumann faces 4 (v=1, x=0 plane,
    dS = du dw), 5/6 (w=0/1, dS = r|c'| du dv), Dirichlet data on sides 1-3 by one joint L2 projection
    (face measures |c'| dv dw on u=0, 2|c'| dv dw on u=1, du dw on v=0; reading N1.a), lifting with the
    full ring operator.  (p+1)-point Gauss per element and direction, fp64."""
    m = n + p
    xg, wg = gauss(p + 1)
    t = np.concatenate([(e + xg) / n for e in range(n)])
    w = np.concatenate([wg / n for _ in range(n)])
    B = eval_basis(p, n, t)
    sp_ = _speed(t)
    # volume: points (u_i, v_j, w_k)
    U, V, W = np.meshgrid(t, t, t, indexing="ij")
    x, y, z, (r, cx, cy, dcx, dcy) = geometry(U, V, W)
    detJ = r * np.sqrt(dcx * dcx + dcy * dcy)
    fv = _f(x, y, z) * detJ * (w[:, None, None] * w[None, :, None] * w[None, None, :])
    Fall = np.einsum("ijk,ia,jb,kc->cba", fv, B, B, B)
    Uf, Wf = np.meshgrid(t, t, indexing="ij")
    ww = w[:, None] * w[None, :]
    # side 4: v = 1 (x = 0), in-face (u, w), dS = du dw; N_b(1) = δ_{b,m−1}
    x4, y4, z4, _ = geometry(Uf, np.ones_like(Uf), Wf)
    g4 = _GN[4](x4, y4, z4) * ww
    Fall[:, m - 1, :] += np.einsum("ik,ia,kc->ca", g4, B, B)
    # sides 5/6: w = 0 / 1, in-face (u, v), dS = r|c'| du dv
    Uf2, Vf2 = np.meshgrid(t, t, indexing="ij")
    for side, cz in ((5, 0), (6, m - 1)):
        x5, y5, z5, (r5, _, _, d5x, d5y) = geometry(Uf2, Vf2, np.full_like(Uf2, 0.0 if side == 5 else 1.0))
        g5 = _GN[side](x5, y5, z5) * r5 * np.sqrt(d5x * d5x + d5y * d5y) * ww
        Fall[cz, :, :] += np.einsum("ij,ia,jb->ba", g5, B, B)
    uD = _ring_projection(p, n, t, w, B, sp_)
    T = weighted_tables(p, n)
    Uc = uD.reshape(m, m, m)  # (c, b, a)

    def apply(Az, Ay, Ax):
        q = np.einsum("ad,cbd->cba", Ax, Uc)
        q = np.einsum("bd,cda->cba", Ay, q)
        return np.einsum("cd,dba->cba", Az, q)

    KU = apply(T["M"], T["B"], T["A"]) + apply(T["M"], T["Dv"], T["C"]) + apply(T["K"], T["B"], T["E"])
    free = free_index_list(3, m, 0b000111)
    return (Fall.ravel() - KU.ravel())[free], uD


def _ring_projection(p, n, t, w, B, sp_):
    """Joint L2 projection of g_D = u on sides 1 (u=0), 2 (u=1), 3 (v=0) of the ring, dense solve."""
    m = n + p
    T = weighted_tables(p, n)
    a, b, c = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    on = (a == 0) | (a == m - 1) | (b == 0)
    dofs = np.sort((a + m * (b + m * c))[on])
    pos = {int(g): k for k, g in enumerate(dofs)}
    Mb = np.zeros((len(dofs), len(dofs)))
    rhs = np.zeros(len(dofs))
    V1, W1 = np.meshgrid(t, t, indexing="ij")
    ww = w[:, None] * w[None, :]
    faces = []
    for side, fixed, scale in ((1, 0, 1.0), (2, m - 1, 2.0)):  # u = 0 / 1: measure r|c'| dv dw, r = 1 / 2
        xx, yy, zz, _ = geometry(np.full_like(V1, 0.0 if side == 1 else 1.0), V1, W1)
        g = exact_u(xx, yy, zz) * scale * _speed(V1) * ww
        Fface = np.einsum("jk,jb,kc->bc", g, B, B)
        faces.append((lambda i0, i1, fx=fixed: fx + m * (i0 + m * i1), scale * T["B"], T["M"], Fface))
    xx, yy, zz, _ = geometry(V1, np.zeros_like(V1), W1)  # v = 0: (u, w), measure du dw
    g = exact_u(xx, yy, zz) * ww
    Fface = np.einsum("ik,ia,kc->ac", g, B, B)
    faces.append((lambda i0, i1: i0 + m * (0 + m * i1), T["M"], T["M"], Fface))
    for gidx, M0, M1, Fface in faces:
        for i0 in range(m):
            for i1 in range(m):
                gi = pos[gidx(i0, i1)]
                rhs[gi] += Fface[i0, i1]
                for j0 in range(max(0, i0 - p), min(m, i0 + p + 1)):
                    for j1 in range(max(0, i1 - p), min(m, i1 + p + 1)):
                        Mb[gi, pos[gidx(j0, j1)]] += M0[i0, j0] * M1[i1, j1]
    uD = np.zeros(m ** 3)
    uD[dofs] = np.linalg.solve(Mb, rhs)
    return uD


def l2_error_full(p: int, n: int, u_free: np.ndarray, uD: np.ndarray) -> float:
    """‖u_h − u‖_{L2(Ω)} on the ring, (p+2)³ Gauss points per element with the map's det J."""
    m = n + p
    coef = uD.copy()
    coef[free_index_list(3, m, 0b000111)] = u_free
    coef = coef.reshape(m, m, m)
    xg, wg = gauss(p + 2)
    t = np.concatenate([(e + xg) / n for e in range(n)])
    w = np.concatenate([wg / n for _ in range(n)])
    Bq = eval_basis(p, n, t)
    uh = np.einsum("ax,zyx->zya", Bq, coef)
    uh = np.einsum("by,zya->zba", Bq, uh)
    uh = np.einsum("cz,zba->cba", Bq, uh)  # (w, v, u)
    Wq, Vq, Uq = np.meshgrid(t, t, t, indexing="ij")
    x, y, z, (r, cx, cy, dcx, dcy) = geometry(Uq, Vq, Wq)
    detJ = r * np.sqrt(dcx * dcx + dcy * dcy)
    err = (uh - exact_u(x, y, z)) ** 2 * detJ
    return float(np.sqrt(np.einsum("c,b,a,cba->", w, w, w, err)))
