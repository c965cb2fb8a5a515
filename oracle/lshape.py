"""The three-patch thick L-shape: conforming multipatch gluing, the stiffness of
the free DOFs and the paper's L-shape data (source, joint L2 Dirichlet projection, Neumann faces).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

Paper passages:
  * multipatch assembly (§2.3): every patch is assembled as a single patch, the patch
    contributions are added into the global matrix through the local→global DOF map, and "the basis
    functions on each interface from each patch are identified as the same global DoF";
  * the L-shaped benchmark: three patches, Dirichlet data on six faces, Neumann on two,
    f = e^x cos z [−2 y cos(xy) + (x²+y²) sin(xy)], g_D = u = e^x sin(xy) cos z, g_N = ∇u·n;
  * Table 2b: the matrix sizes this layout reproduces.

Reading N4.a: the printed union "[0,1]³ ∪ [0,−1]³ ∪ [1,2]³"
has corner-touching cubes, so the L-prism of three unit-cube patches is taken instead:
    A = [0,1]×[0,1]×[0,1] (corner), B = [1,2]×[0,1]×[0,1] (east), C = [0,1]×[1,2]×[0,1] (north),
each with the paper's maximum-regularity B-spline space of degree p on n³ elements (identity
Jacobian: every patch is a translate of the unit cube). Glued, the control lattice is
    {(x, y, z) : 0 ≤ x, y ≤ 2m−2, 0 ≤ z ≤ m−1, not (x ≥ m and y ≥ m)},   m = n + p,
the re-entrant edge x = y = m−1 being shared by all three patches.
Reading N4.b: of the eight faces of the L-prism, the Dirichlet ones are x=0, y=0, x=2 (B's end),
y=2 (C's end), z=0 and z=1; the Neumann ones are the two faces at the re-entrant edge (y=1 on B,
normal +y: g_N = x e^x cos(xy) cos z, the paper's side 6 formula; x=1 on C, normal +x:
g_N = e^x cos z [sin(xy) + y cos(xy)], its side 4 formula).  Three six-face layouts reproduce every
Table 2b size; this one is the one symmetric in the re-entrant corner.

Numbering: all-DOF and free-DOF indices are the lattice points in lexicographic order, x fastest,
then y, then z (free = the lattice minus the Dirichlet faces, same order).

Stiffness: K_all = Σ_{P = A, B, C} S_Pᵀ K_cube S_P with K_cube the all-DOF unit-cube stiffness of
core.assemble (c.4) and S_P the patch's local→global map; entries are summed in patch order A, B, C
((v_A + v_B) + v_C) so the result is reproducible to the bit.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .bspline import element_loop_matrices_1d, eval_basis, gauss
from .core import assemble

PATCHES = ("A", "B", "C")


def patch_offsets(m: int):
    """Lattice offsets (ox, oy) and physical offsets of patches A, B, C."""
    return {"A": ((0, 0), (0.0, 0.0)), "B": ((m - 1, 0), (1.0, 0.0)), "C": ((0, m - 1), (0.0, 1.0))}


def lattice(m: int):
    """(gidx, inside): gidx[z, y, x] = all-DOF index of lattice point (x, y, z) or −1 outside the L."""
    M = 2 * m - 1
    z, y, x = np.meshgrid(np.arange(m), np.arange(M), np.arange(M), indexing="ij")
    inside = ~((x >= m) & (y >= m))
    gidx = -np.ones(inside.shape, dtype=np.int64)
    gidx[inside] = np.arange(int(inside.sum()))
    return gidx, inside


def dirichlet_mask(m: int) -> np.ndarray:
    """mask[z, y, x]: lattice point on a Dirichlet face (reading N4.b)."""
    M = 2 * m - 1
    z, y, x = np.meshgrid(np.arange(m), np.arange(M), np.arange(M), indexing="ij")
    return ((x == 0) | (y == 0) | ((x == M - 1) & (y <= m - 1)) | ((y == M - 1) & (x <= m - 1))
            | (z == 0) | (z == m - 1))


def free_lists(p: int, n: int):
    """(all-DOF indices of the free DOFs ascending, all-DOF indices of the Dirichlet DOFs, N_all)."""
    m = n + p
    gidx, inside = lattice(m)
    dmask = dirichlet_mask(m)
    free = gidx[inside & ~dmask]
    dir_ = gidx[inside & dmask]
    return free, dir_, int(inside.sum())


def n_free(p: int, n: int) -> int:
    """Free-DOF count (Table 2b P:L1566-1575 pins it)."""
    return len(free_lists(p, n)[0])


def patch_map(m: int, P: str) -> np.ndarray:
    """S_P as an index array: local all-DOF index a + m(b + m c) → global all-DOF index."""
    gidx, _ = lattice(m)
    (ox, oy), _ = patch_offsets(m)[P]
    c, b, a = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    return gidx[c, b + oy, a + ox].ravel()


def assemble_all(p: int, n: int) -> sp.csr_matrix:
    """K_all (all lattice DOFs, no elimination): Σ_P S_Pᵀ K_cube S_P, summed in patch order."""
    return _assemble(p, n, restrict_free=False)


def assemble_lshape(p: int, n: int, chunk_rows: int = 1 << 16) -> sp.csr_matrix:
    """K of the free DOFs (Dirichlet DOFs eliminated)."""
    return _assemble(p, n, restrict_free=True, chunk_rows=chunk_rows)


def _assemble(p: int, n: int, restrict_free: bool, chunk_rows: int = 1 << 16) -> sp.csr_matrix:
    """Σ_P S_Pᵀ K_cube S_P over blocks of `chunk_rows` global rows (memory ∝ the block, not the
    whole operator: the k = 96 L-shape has ~10⁹ non-zeros).  Per entry, the values of the patches
    that hold it are summed in patch order, ((0 + v_A) + v_B) + v_C; the union pattern is kept (also
    entries whose sum is 0).  Each S_P is increasing in the local index, so the local rows of a block
    of global rows are a contiguous range of K_cube's rows."""
    m = n + p
    Kc = assemble(3, p, n, dirichlet_sides=0)
    free, _, Nall = free_lists(p, n)
    if restrict_free:
        pos = -np.ones(Nall, dtype=np.int64)
        pos[free] = np.arange(len(free))
    maps = [patch_map(m, P) for P in PATCHES]
    rp, ci, vv, nnz = [np.zeros(1, dtype=np.int64)], [], [], 0
    nrow_out = len(free) if restrict_free else Nall
    for g0 in range(0, Nall, chunk_rows):
        g1 = min(Nall, g0 + chunk_rows)
        keys, vals = [], []
        for g in maps:
            lo, hi = np.searchsorted(g, g0), np.searchsorted(g, g1)
            blk = Kc[lo:hi].tocoo()
            keys.append(g[blk.row + lo] * Nall + g[blk.col])
            vals.append(blk.data)
        ukeys = np.unique(np.concatenate(keys))  # the union pattern of the block, row-major
        v = np.zeros(len(ukeys))
        for k, d in zip(keys, vals):  # ((0 + v_A) + v_B) + v_C
            vp = np.zeros(len(ukeys))
            vp[np.searchsorted(ukeys, k)] = d
            v = v + vp
        rows, cols = ukeys // Nall, ukeys % Nall
        if restrict_free:
            keep = (pos[rows] >= 0) & (pos[cols] >= 0)
            rows, cols, v = pos[rows[keep]], pos[cols[keep]], v[keep]
            r_lo = int(np.searchsorted(free, g0))
            r_hi = int(np.searchsorted(free, g1))
        else:
            r_lo, r_hi = g0, g1
        cnt = np.bincount(rows - r_lo, minlength=r_hi - r_lo)
        rp.append(nnz + np.cumsum(cnt))
        nnz += len(v)
        ci.append(cols.astype(np.int32))
        vv.append(v)
    K = sp.csr_matrix((np.concatenate(vv), np.concatenate(ci), np.concatenate(rp)), shape=(nrow_out, nrow_out))
    K.has_sorted_indices = True
    return K


# ------------------------------------------------------------------------------------------------
# the paper's L-shape data
# ------------------------------------------------------------------------------------------------
def exact_u(x, y, z):
    return np.exp(x) * np.sin(x * y) * np.cos(z)


def source_f(x, y, z):
    return np.exp(x) * np.cos(z) * (-2.0 * np.cos(x * y) * y + np.sin(x * y) * (y * y + x * x))


def gN_side4(x, y, z):  # +x normal
    return np.cos(z) * np.exp(x) * (np.sin(x * y) + y * np.cos(x * y))


def gN_side6(x, y, z):  # +y normal
    return x * np.exp(x) * np.cos(x * y) * np.cos(z)


def _quad_1d(p: int, n: int):
    xg, wg = gauss(p + 1)
    x = np.concatenate([(e + xg) / n for e in range(n)])
    w = np.concatenate([wg / n for _ in range(n)])
    return x, w, eval_basis(p, n, x)


# patch faces: (patch, axis, end, kind) with kind 'D' (Dirichlet), 'N' (Neumann, its g_N) or 'I'
FACES = (
    ("A", 0, 0, "D"), ("A", 0, 1, "I"), ("A", 1, 0, "D"), ("A", 1, 1, "I"), ("A", 2, 0, "D"), ("A", 2, 1, "D"),
    ("B", 0, 0, "I"), ("B", 0, 1, "D"), ("B", 1, 0, "D"), ("B", 1, 1, "N6"), ("B", 2, 0, "D"), ("B", 2, 1, "D"),
    ("C", 0, 0, "D"), ("C", 0, 1, "N4"), ("C", 1, 0, "I"), ("C", 1, 1, "D"), ("C", 2, 0, "D"), ("C", 2, 1, "D"),
)


def _face_values(p, n, P, ax, end, g):
    """(global all-DOF indices of the face DOFs (i0, i1) in-face order, ∫_face g N_i0 N_i1 dS) on patch
    P's face {ξ_ax = end}; the in-face axes are the other two, ascending."""
    m = n + p
    x, w, B = _quad_1d(p, n)
    _, (px, py) = patch_offsets(m)[P]
    fa = [a for a in range(3) if a != ax]
    U, V = np.meshgrid(x, x, indexing="ij")
    pts = [None, None, None]
    pts[ax] = np.full_like(U, float(end))
    pts[fa[0]], pts[fa[1]] = U, V
    gv = g(pts[0] + px, pts[1] + py, pts[2]) * (w[:, None] * w[None, :])
    Fface = np.einsum("uv,ua,vb->ab", gv, B, B)
    i0, i1 = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    loc = [None, None, None]
    loc[ax] = np.full_like(i0, 0 if end == 0 else m - 1)
    loc[fa[0]], loc[fa[1]] = i0, i1
    g_all = patch_map(m, P)[loc[0] + m * (loc[1] + m * loc[2])]
    return g_all, Fface


def load_all(p: int, n: int, f=None, gN4=None, gN6=None) -> np.ndarray:
    """Source + Neumann load on every lattice DOF: Σ_P S_Pᵀ (∫_P f φ + ∫_{∂P ∩ Γ_N} g_N φ)."""
    f = source_f if f is None else f
    gN = {"N4": gN_side4 if gN4 is None else gN4, "N6": gN_side6 if gN6 is None else gN6}
    m = n + p
    _, _, Nall = free_lists(p, n)
    x, w, B = _quad_1d(p, n)
    Fall = np.zeros(Nall)
    for P in PATCHES:
        _, (px, py) = patch_offsets(m)[P]
        X, Y, Z = np.meshgrid(x + px, x + py, x, indexing="ij")
        fv = f(X, Y, Z) * (w[:, None, None] * w[None, :, None] * w[None, None, :])
        Fp = np.einsum("ijk,ia,jb,kc->cba", fv, B, B, B).ravel()
        np.add.at(Fall, patch_map(m, P), Fp)
    for P, ax, end, kind in FACES:
        if kind in ("N4", "N6"):
            g_all, Fface = _face_values(p, n, P, ax, end, gN[kind])
            np.add.at(Fall, g_all.ravel(), Fface.ravel())
    return Fall


def dirichlet_projection(p: int, n: int, gD=None) -> np.ndarray:
    """All-DOF vector with the joint L2 projection of g_D onto the trace space of the union of the
    Dirichlet patch faces (one boundary mass system, reading c.NEXT-1 of the cube applied to the glued
    boundary), 0 elsewhere."""
    m = n + p
    _, dir_, Nall = free_lists(p, n)
    pos = -np.ones(Nall, dtype=np.int64)
    pos[dir_] = np.arange(len(dir_))
    M1, _ = element_loop_matrices_1d(p, n)
    FM = sp.kron(sp.csr_matrix(M1), sp.csr_matrix(M1)).tocoo()  # face mass, (i0 m + i1, j0 m + j1)
    rows, cols, vals = [], [], []
    rhs = np.zeros(len(dir_))
    for P, ax, end, kind in FACES:
        if kind != "D":
            continue
        g_all, Fface = _face_values(p, n, P, ax, end, exact_u if gD is None else gD)
        gf = g_all.ravel()
        rows.append(pos[gf[FM.row]])
        cols.append(pos[gf[FM.col]])
        vals.append(FM.data)
        np.add.at(rhs, pos[gf], Fface.ravel())
    Mb = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                       shape=(len(dir_), len(dir_)))
    uD = np.zeros(Nall)
    uD[dir_] = spla.spsolve(Mb.tocsc(), rhs)
    return uD


def paper_lshape_rhs(p: int, n: int, f=None, gD=None, gN4=None, gN6=None):
    """(F_free, u_D_all): F_free = F_all[free] − (K_all u_D)[free] (lifting).  The data default to the
    paper's; other callables serve the polynomial-reproduction pin."""
    free, _, _ = free_lists(p, n)
    uD = dirichlet_projection(p, n, gD)
    Fall = load_all(p, n, f, gN4, gN6)
    return (Fall - assemble_all(p, n) @ uD)[free], uD


def greville(p: int, n: int) -> np.ndarray:
    """Greville abscissae of the open uniform knot vector on [0, 1] (the coefficients of t ↦ t)."""
    t = np.concatenate([np.zeros(p), np.linspace(0.0, 1.0, n + 1), np.ones(p)])
    return np.array([t[a + 1:a + p + 1].mean() for a in range(n + p)])


def lattice_coords(p: int, n: int):
    """Physical (x, y, z) Greville coordinates of every lattice DOF, all-DOF order."""
    m = n + p
    gidx, inside = lattice(m)
    gr = greville(p, n)
    # lattice index i along x: patch-local a = i (i ≤ m−1) or a = i − (m−1) shifted by 1
    ext = np.concatenate([gr, 1.0 + gr[1:]])
    z, y, x = np.meshgrid(np.arange(m), np.arange(2 * m - 1), np.arange(2 * m - 1), indexing="ij")
    return ext[x[inside]], ext[y[inside]], gr[z[inside]]


def l2_error_full(p: int, n: int, u_free: np.ndarray, uD: np.ndarray, exact=None) -> float:
    """‖u_h − u‖_{L2(Ω)}, u_h = free part + Dirichlet part, (p+2)³ Gauss points per element per patch."""
    m = n + p
    free, _, _ = free_lists(p, n)
    coef = uD.copy()
    coef[free] = u_free
    xg, wg = gauss(p + 2)
    pts = np.concatenate([(e + xg) / n for e in range(n)])
    wts = np.concatenate([wg / n for _ in range(n)])
    B = eval_basis(p, n, pts)
    err = 0.0
    for P in PATCHES:
        _, (px, py) = patch_offsets(m)[P]
        c = coef[patch_map(m, P)].reshape(m, m, m)
        uh = np.einsum("ax,zyx->zya", B, c)
        uh = np.einsum("by,zya->zba", B, uh)
        uh = np.einsum("cz,zba->cba", B, uh)
        Zq, Yq, Xq = np.meshgrid(pts, pts + py, pts + px, indexing="ij")
        err += float(np.einsum("c,b,a,cba->", wts, wts, wts, (uh - (exact_u if exact is None else exact)(Xq, Yq, Zq)) ** 2))
    return float(np.sqrt(err))
