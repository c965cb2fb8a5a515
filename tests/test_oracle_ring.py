"""Pins of the oracle's thick-quarter-ring operator (PAPER.md P:L1091-1102,
non-isoparametric entries P:L598-603, Table 3).

* the separable route (weighted 1-D tables, Kronecker sum) equals a genuine 3-D element loop that
  applies J⁻¹J⁻ᵀ det J of the NURBS map at every Gauss point (independent route);
* sizes equal Table 3b; K symmetric (bitwise) and SPD; with no Dirichlet side K·1 = 0;
* Σ (E_u ⊗ B_v ⊗ M_w) = ∫ det J = |Ω| = 3π/4 up to the quadrature error;
* the hierarchy's operator complexity reproduces Table 3c within ±0.02 (the c.12 reading on a second
  geometry).
"""
import numpy as np
import pytest

import oracle
from oracle import ring

TABLE3B = {(12, 2): 2184, (12, 3): 2730, (12, 4): 3360, (12, 5): 4080,
           (24, 2): 15600, (24, 3): 17550, (24, 4): 19656, (24, 5): 21924}
TABLE3C = {(12, 2): 1.22, (12, 3): 1.15, (24, 2): 1.34, (24, 3): 1.23, (24, 4): 1.18}


@pytest.mark.parametrize("p,n", [(2, 3), (3, 2), (2, 4)])
def test_separable_route_equals_3d_element_loop(p, n):
    K = ring.assemble_ring(p, n).toarray()
    Kd = ring.element_loop_ring(p, n)
    assert np.abs(K - Kd).max() <= 1e-13 * np.abs(Kd).max()


@pytest.mark.parametrize("k,p", sorted(TABLE3B))
def test_sizes_table3b(k, p):
    """Table 3b: the number of free DOFs of the ring operator the oracle assembles
    (its Dirichlet sides eliminated, R.a) equals the printed size."""
    K = ring.assemble_ring(p, k)
    assert K.shape == (TABLE3B[(k, p)], TABLE3B[(k, p)])


def test_symmetric_spd_and_neumann_kernel():
    K = ring.assemble_ring(3, 4)
    assert (K != K.T).nnz == 0
    np.linalg.cholesky(K.toarray())
    Kn = ring.assemble_ring(3, 4, dirichlet_sides=0)
    assert np.abs(Kn @ np.ones(Kn.shape[0])).max() <= 1e-13 * abs(Kn).max()


def test_volume():
    T = ring.weighted_tables(3, 8)
    vol = T["E"].sum() * T["B"].sum() * T["M"].sum()
    assert abs(vol - 3 * np.pi / 4) <= 1e-6 * 3 * np.pi / 4


@pytest.mark.parametrize("k,p", sorted(TABLE3C))
def test_operator_complexity_table3c(k, p):
    H = oracle.setup(ring.assemble_ring(p, k), oracle.OParams.for_degree(p))
    assert abs(H.opc() - TABLE3C[(k, p)]) <= 0.02, H.opc()


@pytest.mark.parametrize("p", [2, 3])
def test_paper_ring_data_converges_at_order(p):
    """The paper's ring problem (u = e^x sin(xy) cos z) with its projected Dirichlet and
    Neumann data: L2 error decays at rate ≥ p + 0.5 under refinement (n = 4, 8, 12)."""
    import scipy.sparse.linalg as spla
    ns = (4, 8, 12)
    errs = []
    for n in ns:
        F, uD = ring.paper_ring_rhs(p, n)
        uf = spla.spsolve(ring.assemble_ring(p, n).tocsc(), F)
        errs.append(ring.l2_error_full(p, n, uf, uD))
    rates = [np.log(errs[i] / errs[i + 1]) / np.log(ns[i + 1] / ns[i]) for i in range(2)]
    assert min(rates) >= p + 0.5, (errs, rates)
