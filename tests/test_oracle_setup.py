"""Pins of the oracle's setup (c.6-c.15): weights, matching, aggregates, prolongators, Galerkin
operators, OPC — against toy values, brute force, hand-derived worked examples, dense algebra and
the paper's Table 1c."""
import itertools
import math

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle import bspline


# --- c.7: compatibility weights (eq:cij) -------------------------------------------

def test_cij_toy_values():
    """K=[[2,−1],[−1,2]]: w=(1,1) → 1.5; w=(1,−1) → 0.5; k_ij=0 → 1."""
    assert oracle.cij(-1.0, 2.0, 2.0, 1.0, 1.0) == 1.5
    assert oracle.cij(-1.0, 2.0, 2.0, 1.0, -1.0) == 0.5
    assert oracle.cij(0.0, 2.0, 2.0, 1.0, 1.0) == 1.0


def test_cij_in_open_interval_for_spd_blocks():
    """For an SPD 2×2 block, |k_ij| < sqrt(k_ii k_jj) ⇒ c_ij ∈ (0, 2) for every w."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        kii, kjj = rng.uniform(0.1, 5, 2)
        kij = rng.uniform(-0.999, 0.999) * math.sqrt(kii * kjj)
        wi, wj = rng.uniform(-3, 3, 2)
        c = oracle.cij(kij, kii, kjj, wi, wj)
        assert 0.0 < c < 2.0


# --- c.8: matching (eq:maxprod) ----------------------------------------------------

def weights_to_matrix(n, wts):
    """A matrix whose c_ij with w=1 and unit diagonal equal the given weights: c = 1 − k_ij."""
    A = np.eye(n)
    for (i, j), c in wts.items():
        A[i, j] = A[j, i] = 1.0 - c
    return sp.csr_matrix(A)


def test_spec_path_examples():
    """4-path (0,1):1.5,(1,2):1.2,(2,3):1.5 → {(0,1),(2,3)};
    3-path (0,1):2.0,(1,2):1.5 → (0,1) + singleton 2; all weights ≤ 1 → no pairs."""
    A = weights_to_matrix(4, {(0, 1): 1.5, (1, 2): 1.2, (2, 3): 1.5})
    mate, agg, pv, wn = oracle.pairwise(A, np.ones(4))
    assert list(mate) == [1, 0, 3, 2] and list(agg) == [0, 0, 1, 1]
    A = weights_to_matrix(3, {(0, 1): 2.0, (1, 2): 1.5})
    mate, agg, _, _ = oracle.pairwise(A, np.ones(3))
    assert list(mate) == [1, 0, -1] and list(agg) == [0, 0, 1]
    A = weights_to_matrix(3, {(0, 1): 0.9, (1, 2): 1.0})
    mate, agg, _, _ = oracle.pairwise(A, np.ones(3))
    assert list(mate) == [-1, -1, -1] and list(agg) == [0, 1, 2]


def brute_force_max_product(n, wts):
    """Exhaustive maximum-product matching over eligible edges (c > 1)."""
    edges = [e for e, c in wts.items() if c > 1.0]
    best = 1.0

    def rec(k, used, prod):
        nonlocal best
        best = max(best, prod)
        for t in range(k, len(edges)):
            i, j = edges[t]
            if i not in used and j not in used:
                rec(t + 1, used | {i, j}, prod * wts[(i, j)])
    rec(0, frozenset(), 1.0)
    return best


def locally_dominant(n, wts):
    """The pointer (locally-dominant) algorithm: repeatedly match mutual heaviest eligible pairs,
    heaviness by (c desc, then (min,max) index asc). Independent of the oracle's global sort."""
    adj = {i: [] for i in range(n)}
    for (i, j), c in wts.items():
        if c > 1.0:
            adj[i].append((j, c))
            adj[j].append((i, c))
    mate = [-1] * n

    def best(i):
        cand = [(-c, min(i, j), max(i, j), j) for j, c in adj[i] if mate[j] < 0]
        return min(cand)[3] if cand else -1
    changed = True
    while changed:
        changed = False
        ptr = [best(i) if mate[i] < 0 else -1 for i in range(n)]
        for i in range(n):
            j = ptr[i]
            if j >= 0 and ptr[j] == i and i < j:
                mate[i], mate[j] = j, i
                changed = True
    return mate


@pytest.mark.parametrize("seed", range(40))
def test_matching_vs_brute_force_and_locally_dominant(seed):
    """Greedy = the unique locally-dominant matching (c.8), and it is a ½-approximation of the
    maximum of Σ log c (i.e. product ≥ sqrt(optimal product)) — checked by exhaustive search."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(4, 11))
    wts = {}
    for i, j in itertools.combinations(range(n), 2):
        if rng.random() < 0.5:
            wts[(i, j)] = float(rng.choice([0.8, 1.1, 1.25, 1.5, 1.5, 1.9]))  # many ties
    A = weights_to_matrix(n, wts)
    mate, agg, pv, wn = oracle.pairwise(A, np.ones(n))
    assert list(mate) == locally_dominant(n, wts)
    prod = 1.0
    for i in range(n):
        if mate[i] > i:
            prod *= wts[(i, int(mate[i]))]
    assert prod >= math.sqrt(brute_force_max_product(n, wts)) * (1 - 1e-12)


# --- c.9/c.11: aggregates and tentative prolongators (eq:prolongation) -------------

def test_pairwise_prolongator_orthonormal_and_numbering():
    K = oracle.assemble(2, 2, 8)
    rng = np.random.default_rng(3)
    w = rng.uniform(0.5, 2.0, K.shape[0])
    mate, agg, pv, wn = oracle.pairwise(K, w)
    n, nc = K.shape[0], wn.size
    P = sp.csr_matrix((pv, (np.arange(n), agg)), shape=(n, nc))
    assert np.abs((P.T @ P).toarray() - np.eye(nc)).max() <= 1e-15
    assert np.abs(P.T @ w - wn).max() <= 1e-14 * wn.max()
    # aggregates numbered in ascending order of their minimum member (c.9)
    first = [np.flatnonzero(agg == I).min() for I in range(nc)]
    assert first == sorted(first)
    # pairs are matched edges of the graph
    for i in range(n):
        if mate[i] >= 0:
            assert mate[mate[i]] == i and K[i, mate[i]] != 0


def test_singleton_value_is_sign():
    """singleton with w_s = −2 → entry −1 (w/|w|)."""
    A = sp.csr_matrix(np.eye(2))
    mate, agg, pv, wn = oracle.pairwise(A, np.array([-2.0, 3.0]))
    assert list(pv) == [-1.0, 1.0] and list(wn) == [2.0, 3.0]


# --- c.12/c.13: smoothed prolongator and Galerkin operator -------------------------------------

def test_worked_example_1d_laplacian():
    """Hand-derived: K = tridiag(−1,2,−1), N=4, w=1, one pairwise step (θ=0.01 keeps every entry).
    All c_ij = 1.5 (tie) → pairs (0,1),(2,3) by index; λ̂ = ‖D⁻¹K‖∞ = 4/2 = 2 ⇒ ω = 2/3;
    P = [[1,0],[1,0],[0,1],[0,1]]/√2, KP = [[1,0],[1,−1],[−1,1],[0,1]]/√2,
    P̄ = P − (ω/2)·KP = [[2/3,0],[2/3,1/3],[1/3,2/3],[0,2/3]]/√2."""
    K = sp.csr_matrix(np.array([[2., -1, 0, 0], [-1, 2, -1, 0], [0, -1, 2, -1], [0, 0, -1, 2]]))
    H = oracle.setup(K, oracle.OParams(agg_steps=1, coarse_size=2, cheb_degree=2))
    L0 = H.levels[0]
    assert list(L0.agg) == [0, 0, 1, 1]
    assert L0.omega == pytest.approx(2.0 / 3.0, rel=1e-15)
    expect = np.array([[2 / 3, 0], [2 / 3, 1 / 3], [1 / 3, 2 / 3], [0, 2 / 3]]) / math.sqrt(2)
    assert np.abs(L0.P.toarray() - expect).max() <= 1e-15
    Kc = expect.T @ K.toarray() @ expect
    assert np.abs(H.levels[1].K.toarray() - Kc).max() <= 1e-15


def _random_mmatrix(n: int, seed: int) -> sp.csr_matrix:
    """A sparse SPD matrix with random negative couplings (no two c_ij equal, so round-off in the
    check cannot flip a tie): graph Laplacian of a random graph + a random positive shift."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in rng.choice(n, size=4, replace=False):
            if j != i:
                v = -rng.uniform(0.2, 2.0)
                rows += [i, j]
                cols += [j, i]
                vals += [v, v]
    A = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    A.sum_duplicates()
    A = A + sp.diags(-np.asarray(A.sum(axis=1)).ravel() + rng.uniform(0.01, 0.1, n))
    return sp.csr_matrix(A)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_intermediate_galerkin_c10_dense_and_step2_matching(seed):
    """c.10 pinned directly: the intermediate operator of one pairwise step equals the
    dense sym(P₁ᵀAP₁) (numpy matmul, an independent route) to round-off; the second matching step
    run on that dense operator gives the aggregates a 2-step setup builds (composition of the two
    steps); and the pattern is the structural pattern of P₁ᵀ|A|P₁."""
    A = _random_mmatrix(300, seed)
    w = np.ones(A.shape[0])  # w⁽⁰⁾ = 1 (c.6), as the setup below starts
    mate, agg1, pv1, wn1 = oracle.pairwise(A, w)
    nc = wn1.size
    assert nc < A.shape[0]
    Ac = oracle.galerkin_pairwise(A, agg1, pv1, nc)
    P1 = np.zeros((A.shape[0], nc))
    P1[np.arange(A.shape[0]), agg1] = pv1
    G = P1.T @ A.toarray() @ P1
    G = 0.5 * (G + G.T)
    assert np.abs(Ac.toarray() - G).max() <= 1e-14 * np.abs(G).max()
    pat = (np.abs(P1).T @ np.abs(A.toarray()) @ np.abs(P1)) > 0
    Acs = Ac.copy()
    Acs.data[:] = 1.0
    assert np.array_equal(Acs.toarray() != 0, pat)  # stored pattern = structural P₁ᵀ|A|P₁
    # step 2 on the dense operator (stored with the same pattern) with the carried test vector w₁
    Gs = sp.csr_matrix(np.where(pat, G, 0.0))
    mate2, agg2, pv2, wn2 = oracle.pairwise(Gs, wn1)
    H = oracle.setup(A, oracle.OParams(agg_steps=2, smooth_prolong=0, coarse_size=1, max_levels=2,
                                       cheb_degree=2))
    L0 = H.levels[0]
    assert np.array_equal(L0.agg, agg2[agg1])
    assert np.allclose(L0.ptent, pv1 * pv2[agg1], rtol=1e-14, atol=0)
    assert H.levels[1].N == wn2.size


@pytest.fixture(scope="module")
def c1_hier():
    K = oracle.assemble(2, 2, 16)
    return K, oracle.setup(K, oracle.OParams.for_degree(2))


def test_c1_hierarchy_galerkin_dense(c1_hier):
    """c.13: K_{l+1} = sym(P̄ᵀ K_l P̄) against dense algebra; R = P̄ᵀ; SPD by Cholesky."""
    K, H = c1_hier
    assert H.levels[0].N == 272  # (n+p-2)(n+p-1) for n=16, p=2
    for l in range(H.nlevels - 1):
        Ll, Lc = H.levels[l], H.levels[l + 1]
        P = Ll.P.toarray()
        assert (Ll.R != Ll.P.T).nnz == 0
        G = P.T @ Ll.K.toarray() @ P
        G = 0.5 * (G + G.T)
        assert np.abs(Lc.K.toarray() - G).max() <= 1e-13 * np.abs(G).max()
        assert (Lc.K != Lc.K.T).nnz == 0
        np.linalg.cholesky(Lc.K.toarray())


def test_tentative_composite_orthonormal(c1_hier):
    """c.11: composite tentative P has one entry per row and PᵀP = I; aggregates ≤ 2^3 = 8."""
    K, H = c1_hier
    L0 = H.levels[0]
    nc = H.levels[1].N
    P = sp.csr_matrix((L0.ptent, (np.arange(L0.N), L0.agg)), shape=(L0.N, nc))
    assert np.abs((P.T @ P).toarray() - np.eye(nc)).max() <= 1e-14
    assert np.bincount(L0.agg).max() <= 8
    assert nc >= math.ceil(L0.N / 8)


def test_smoothed_prolongator_keeps_near_kernel(c1_hier):
    """c.12: on rows where (K w)_i = 0 the filtered smoothing term vanishes (lumping preserves row
    sums), so P̄ w_c = w there; and the dense formula P̄ = P − ω D_f⁻¹ K_f P holds with θ=0."""
    K, H = c1_hier
    L0, L1 = H.levels[0], H.levels[1]
    Kw = K @ L0.w
    rows = np.abs(Kw) <= 1e-12 * np.abs(K.diagonal()).max()
    assert rows.sum() > 50
    assert np.abs((L0.P @ L1.w)[rows] - L0.w[rows]).max() <= 1e-12
    Hu = oracle.setup(K, oracle.OParams.for_degree(2, filter_theta=0.0))
    L0u = Hu.levels[0]
    nc = Hu.levels[1].N
    Pt = sp.csr_matrix((L0u.ptent, (np.arange(L0u.N), L0u.agg)), shape=(L0u.N, nc)).toarray()
    Kd = K.toarray()
    D = np.diag(Kd)
    lam = (np.abs(Kd).sum(axis=1) / D).max()
    om = 4.0 / (3.0 * lam)
    Pbar = Pt - om * (Kd @ Pt) / D[:, None]
    assert L0u.omega == pytest.approx(om, rel=1e-14)
    assert np.abs(L0u.P.toarray() - Pbar).max() <= 1e-14


def test_l1_diagonal(c1_hier):
    """c.15: d̂_i = Σ_j |k_ij| > 0 and λ_max(D̂⁻¹K) ≤ 1 (Gershgorin)."""
    K, H = c1_hier
    for L in H.levels:
        Kd = L.K.toarray()
        assert np.allclose(L.dhat, np.abs(Kd).sum(axis=1), rtol=1e-15, atol=0)
        s = 1.0 / np.sqrt(L.dhat)
        lam = np.linalg.eigvalsh(s[:, None] * Kd * s[None, :])
        assert lam.max() <= 1.0 + 1e-13 and lam.min() > 0


@pytest.mark.parametrize("k,p", [(24, 3), (24, 4), (24, 5), pytest.param(48, 3, marks=pytest.mark.slow)])
def test_opc_table1c(table1, k, p):
    """PAPER pin, Table 1c: operator complexity within ±0.02 at k ≥ 24 under the
    c.12 reading (θ = 0.01 filtered smoothing matrix, ω = 4/(3‖D_f⁻¹K_f‖∞))."""
    K = oracle.assemble(3, p, k)
    H = oracle.setup(K, oracle.OParams.for_degree(p))
    assert abs(H.opc() - table1[(k, p)][1]) <= 0.02, H.opc()
    assert H.levels[-1].N <= 50 and H.levels[-2].N > 50


def _study():
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "oracle", "opc_study.json")) as f:
        st = json.load(f)
    with open(os.path.join(root, "oracle", "sizes_C3.json")) as f:
        c3 = json.load(f)
    st["k96_p3"]["canonical"] = dict(opc=c3["opc"], N=c3["N"])
    return st


def test_opc_tie_order_study(table1):
    """PAPER pin of the tie-order reading (DESIGN.md c.8t) on the committed study (written by the
    oracle-only oracle/scripts/opc_study.py; oracle/sizes_C3.json for the canonical k = 96 setup):
    Table 1c at (24,3), (48,3), (96,3) and (96,4) lies between the two kinds of tie order — the
    pseudo-random order (3 seeds) within ±0.015 of the paper (printed to 2 decimals) at every k, the
    index orders (canonical, and preferring the larger index) at most 0.035 below it and never above
    it by more than 0.005."""
    st = _study()
    for k in (24, 48, 96):
        paper = table1[(k, 3)][1]
        r = st[f"k{k}_p3"]
        hashed = [v["opc"] for n, v in r.items() if n.startswith("tie_hashed")]
        assert hashed and all(abs(h - paper) <= 0.015 for h in hashed), (k, hashed, paper)
        assert max(hashed) - min(hashed) <= 0.002
        for n in ("canonical", "tie_larger_index"):
            assert paper - 0.035 <= r[n]["opc"] <= paper + 0.005, (k, n, r[n]["opc"], paper)
        assert r["canonical"]["N"][0] == table1[(k, 3)][0]
    # (96,4): the same picture with a wider tie spread at p = 4 (1.258 index order, 1.301 pseudo-random,
    # paper 1.30)
    r, paper = st["k96_p4"], table1[(96, 4)][1]
    assert abs(r["tie_hashed"]["opc"] - paper) <= 0.015, r["tie_hashed"]["opc"]
    assert paper - 0.045 <= r["canonical"]["opc"] <= paper + 0.005, r["canonical"]["opc"]
    assert r["canonical"]["N"][0] == table1[(96, 4)][0]


@pytest.mark.slow
def test_opc_table1c_k96(table1):
    """Table 1c at the headline size (96,3), recomputed (~5 min, ~15 GB): the pseudo-random tie order
    reproduces the paper's 1.34 within ±0.01 (the canonical index order: `test_opc_tie_order_study`)."""
    K = oracle.assemble(3, 3, 96)
    H = oracle.setup(K, oracle.OParams.for_degree(3, tie_break=2))
    assert abs(H.opc() - table1[(96, 3)][1]) <= 0.01, H.opc()
    assert H.levels[0].N == table1[(96, 3)][0]


def test_setup_deterministic(c1_hier):
    K, H = c1_hier
    H2 = oracle.setup(K, oracle.OParams.for_degree(2))
    for a, b in zip(H.levels, H2.levels):
        assert (a.K != b.K).nnz == 0 and np.array_equal(a.K.data, b.K.data)
