"""Pins of the oracle's solve phase (c.16-c.19) against closed forms and dense algebra."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl

import oracle
from oracle import bspline
import amg_inputs


def dense_smoother(Kd, dhat, m):
    """x = S b for the 4th-kind Chebyshev smoother from x0 = 0, from its closed-form error polynomial
    E_m = W_m(I − 2 D̂⁻¹K)/(2m+1) with W_m(cos θ) = sin((m+½)θ)/sin(θ/2) (Lottes), so
    S = (I − E_m) K⁻¹.  Computed by eigendecomposition of D̂^{-1/2} K D̂^{-1/2}."""
    s = 1.0 / np.sqrt(dhat)
    G = s[:, None] * Kd * s[None, :]
    lam, Q = np.linalg.eigh(G)
    th = np.arccos(np.clip(1.0 - 2.0 * lam, -1.0, 1.0))
    f = np.sin((m + 0.5) * th) / np.sin(0.5 * th) / (2 * m + 1)
    E = (s[:, None] * (Q * f) @ Q.T) / s[None, :]  # D^{-1/2} Q f Qᵀ D^{1/2}
    n = Kd.shape[0]
    return (np.eye(n) - E) @ np.linalg.inv(Kd)


@pytest.fixture(scope="module")
def c1():
    K = oracle.assemble(2, 2, 16)
    H = oracle.setup(K, oracle.OParams.for_degree(2))
    return K, H


@pytest.mark.parametrize("m", [1, 2, 4, 8])
def test_chebyshev_smoother_polynomial(c1, m):
    """c.16: the recurrence equals the closed-form 4th-kind polynomial; degree 1 ⇒ I − (4/3)D̂⁻¹K."""
    K, _ = c1
    H = oracle.setup(K, oracle.OParams(cheb_degree=m, agg_steps=3))
    L0 = H.levels[0]
    Kd = K.toarray()
    S = dense_smoother(Kd, L0.dhat, m)
    rng = np.random.default_rng(m)
    b = rng.uniform(-1, 1, K.shape[0])
    x = oracle.smooth(H, 0, b)
    assert np.abs(x - S @ b).max() <= 1e-11 * np.abs(S @ b).max()
    if m == 1:
        assert np.allclose(x, (4.0 / 3.0) * b / L0.dhat, rtol=1e-15, atol=0)
    # x* is a fixed point: S(K x*, x*) = x*
    xs = rng.uniform(-1, 1, K.shape[0])
    assert np.abs(oracle.smooth(H, 0, K @ xs, xs) - xs).max() <= 1e-12


def test_coarse_solve_is_jacobi_series(c1):
    """c.17: 30 ℓ1-Jacobi sweeps from 0 equal Σ_{k<30} (I − D̂⁻¹K)^k D̂⁻¹ b (a one-level hierarchy's V-cycle)."""
    K, _ = c1
    H = oracle.setup(K, oracle.OParams(coarse_size=10 ** 6))
    assert H.nlevels == 1
    b = np.random.default_rng(1).uniform(-1, 1, K.shape[0])
    d = H.levels[0].dhat
    Kd = K.toarray()
    x = np.zeros_like(b)
    term = b / d
    for _ in range(30):
        x = x + term
        term = term - (Kd @ term) / d
    y = oracle.vcycle(H, b)
    assert np.abs(y - x).max() <= 1e-12 * np.abs(x).max()


def test_two_grid_dense_formula(c1):
    """c.18: the oracle's 2-level V-cycle equals the dense composition
    x1 = S b; e = C R (b − K x1); x2 = x1 + P̄ e; x = x2 + S (b − K x2), with S from the closed-form
    polynomial and C the closed-form Jacobi series on the coarse level."""
    K, H = c1
    assert H.nlevels == 2
    L0, L1 = H.levels
    Kd, Kc = K.toarray(), L1.K.toarray()
    S = dense_smoother(Kd, L0.dhat, H.prm.cheb_degree)
    nc = L1.N
    C = np.zeros((nc, nc))
    T = np.diag(1.0 / L1.dhat)
    for _ in range(30):
        C += T
        T = T - (Kc @ T) / L1.dhat[:, None]
    P = L0.P.toarray()
    b = np.random.default_rng(2).uniform(-1, 1, K.shape[0])
    x1 = S @ b
    x2 = x1 + P @ (C @ (P.T @ (b - Kd @ x1)))
    x = x2 + S @ (b - Kd @ x2)
    y = oracle.vcycle(H, b)
    assert np.abs(y - x).max() <= 1e-11 * np.abs(x).max()


@pytest.mark.parametrize("case", [(2, 2, 16), (3, 3, 12)])
def test_vcycle_symmetric(case):
    """⟨V r1, r2⟩ = ⟨r1, V r2⟩ (R = P̄ᵀ, post = pre) and ⟨V r, r⟩ > 0."""
    K = oracle.assemble(*case)
    H = oracle.setup(K, oracle.OParams.for_degree(case[1]))
    rng = np.random.default_rng(5)
    r1, r2 = rng.uniform(-1, 1, (2, K.shape[0]))
    a, b = oracle.vcycle(H, r1) @ r2, r1 @ oracle.vcycle(H, r2)
    assert abs(a - b) <= 1e-12 * max(abs(a), abs(b))
    assert oracle.vcycle(H, r1) @ r1 > 0


def test_pcg_identity_preconditioner_is_cg_exact_on_2x2():
    """c.19 with a one-level hierarchy of a 2×2 SPD system: PCG terminates in ≤ 2 iterations with
    the exact solution (finite termination of CG in exact arithmetic)."""
    K = sp.csr_matrix(np.array([[4.0, 1.0], [1.0, 3.0]]))
    H = oracle.setup(K, oracle.OParams(coarse_size=10))
    F = np.array([1.0, 2.0])
    u, it, rr, hist, rc = oracle.pcg(H, F, rtol=1e-14, maxit=10)
    assert rc == 0 and it <= 2
    assert np.abs(u - np.linalg.solve(K.toarray(), F)).max() <= 1e-14


def test_pcg_zero_rhs(c1):
    """F = 0 → u = 0, 0 iterations."""
    K, H = c1
    u, it, rr, hist, rc = oracle.pcg(H, np.zeros(K.shape[0]))
    assert it == 0 and rc == 0 and not u.any()


def test_pcg_converges_to_direct_solution_and_energy_decreases(c1):
    """c.19: converged u satisfies the true residual bound and matches the direct solve; the energy
    norm of the error decreases monotonically."""
    K, H = c1
    F = bspline.load_vector(2, 2, 16)
    ustar = spl.spsolve(K.tocsc(), F)
    u, it, rr, hist, rc = oracle.pcg(H, F, rtol=1e-6)
    assert rc == 0 and 1 <= it <= 20
    assert np.linalg.norm(F - K @ u) <= 1.01e-6 * np.linalg.norm(F)
    assert rr <= 1e-6 and hist[0] == 1.0
    en = []
    for k in range(1, it + 1):
        uk = oracle.pcg(H, F, rtol=0.0, maxit=k)[0]
        e = uk - ustar
        en.append(e @ (K @ e))
    assert all(en[i + 1] < en[i] for i in range(len(en) - 1))
    assert np.linalg.norm(u - ustar) <= 1e-4 * np.linalg.norm(ustar)


def test_pcg_deterministic(c1):
    K, H = c1
    F = np.random.default_rng(9).uniform(-1, 1, K.shape[0])
    a = oracle.pcg(H, F)
    b = oracle.pcg(H, F)
    assert a[1] == b[1] and np.array_equal(a[0], b[0])


# --- NEXT-1 solvers: §5.1 coarse CG and the flexible outer CG ------------------
def test_coarse_cg_finite_termination():
    """Coarse solver 1 (CG preconditioned by one weighted-Jacobi sweep) with tolerance 0 and N
    iterations reaches K⁻¹b (CG finite termination); with the paper's 1e-4 it meets that tolerance."""
    import scipy.sparse.linalg as spla  # noqa: F401
    K = oracle.assemble(2, 2, 4)
    N = K.shape[0]
    b = amg_inputs.uniform_pm1(N, seed=21)
    H = oracle.setup(K, oracle.OParams(cheb_degree=4, coarse_size=10 ** 6, coarse_solver=1, coarse_tol=0.0,
                                       coarse_maxit=N))
    assert H.nlevels == 1
    x = oracle.vcycle(H, b)
    xs = np.linalg.solve(K.toarray(), b)
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)
    H2 = oracle.setup(K, oracle.OParams(cheb_degree=4, coarse_size=10 ** 6, coarse_solver=1))
    x2 = oracle.vcycle(H2, b)
    assert np.linalg.norm(b - K @ x2) <= 1e-4 * np.linalg.norm(b)


@pytest.mark.parametrize("case", [(2, 2, 16), (3, 3, 6)])
def test_fcg_equals_pcg_for_a_fixed_preconditioner(case):
    """With the linear SPD V-cycle (ℓ1-Jacobi coarse sweeps) Notay's FCG(1) — a different α and β —
    generates the CG iterates: same iteration count, same solution to round-off."""
    dim, p, n = case
    K = oracle.assemble(dim, p, n)
    F = amg_inputs.uniform_pm1(K.shape[0], seed=22)
    H = oracle.setup(K, oracle.OParams.for_degree(p))
    u1, it1, rr1, h1, rc1 = oracle.pcg(H, F, rtol=1e-8)
    u2, it2, rr2, h2, rc2 = oracle.fcg(H, F, rtol=1e-8)
    assert rc1 == rc2 == 0 and abs(it1 - it2) <= 1
    assert np.linalg.norm(u1 - u2) <= 1e-7 * np.linalg.norm(u1)
    k = min(len(h1), len(h2))
    assert np.allclose(h1[:k], h2[:k], rtol=1e-5)


def test_fcg_with_the_variable_coarse_cg_is_a_descent_method():
    """With the §5.1 coarse CG (a nonlinear preconditioner) FCG still reduces the energy norm of the
    error monotonically (α minimises along p) and converges."""
    K = oracle.assemble(3, 3, 6)
    F = amg_inputs.uniform_pm1(K.shape[0], seed=23)
    us = np.linalg.solve(K.toarray(), F)
    H = oracle.setup(K, oracle.OParams.for_degree(3, coarse_solver=1))
    energies = []
    for k in range(1, 12):
        u, it, rr, h, rc = oracle.fcg(H, F, rtol=0.0, maxit=k)
        e = u - us
        energies.append(float(e @ (K @ e)))
    assert all(b <= a * (1 + 1e-12) for a, b in zip(energies, energies[1:]))
    u, it, rr, h, rc = oracle.fcg(H, F, rtol=1e-6)
    assert rc == 0 and np.linalg.norm(F - K @ u) <= 1.01e-6 * np.linalg.norm(F)
