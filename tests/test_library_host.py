"""CPU tests of the product library's host side: C-ABI symbols, error behaviour, and BITWISE parity of
the generator and the hierarchy setup with the oracle (DESIGN.md §3 canonical arithmetic contract).

The library and the oracle share no code; both follow the readings c.1-c.15.  The oracle is pinned
separately (tests/test_oracle_*.py)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from oracle import tables
import paper_2511_21268_b200 as amg
from paper_2511_21268_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "amg_b200.h")).read()
    declared = set(re.findall(r"\b(amg_[a-z_]+)\s*\(", hdr)) - {"amg_alloc_fn", "amg_free_fn"}
    declared = {d for d in declared if not d.endswith("_fn")}
    L = _lib.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(_lib.EXPORTED)
    # the checked build (device-side invariant checks, tests/test_gpu_checked.py) exports the same ABI
    chk = os.path.join(ROOT, "paper_2511_21268_b200", "libamg_b200_checked.so")
    if os.path.exists(chk):
        Lc = C.CDLL(chk)
        for name in sorted(declared):
            assert hasattr(Lc, name), name


def test_errors_are_reported_not_raised_through_abi():
    d = _lib.amg_iga_desc(4, 2, 8, 7, 0)
    Kp = C.POINTER(_lib.amg_csr)()
    Fp = C.POINTER(C.c_double)()
    st = _lib.lib().amg_iga_poisson(C.byref(d), C.byref(Kp), C.byref(Fp))
    assert st == -1 and b"dim" in _lib.lib().amg_last_error()
    with pytest.raises(amg.AmgError):
        amg.params(0)
    # non-symmetric K is rejected
    import scipy.sparse as sp
    A = sp.csr_matrix(np.array([[2.0, -1.0], [-0.5, 2.0]]))
    with pytest.raises(amg.AmgError, match="symmetric"):
        amg.Hierarchy(A, amg.params(2, host_only=1))
    # non-positive diagonal
    A = sp.csr_matrix(np.array([[0.0, -1.0], [-1.0, 2.0]]))
    with pytest.raises(amg.AmgError, match="ENOTSPD"):
        amg.Hierarchy(A, amg.params(2, host_only=1))


def test_setup_take_equals_setup():
    """amg_setup_take (the hierarchy takes the generator's arrays over, no copy of K) builds bitwise the
    hierarchy amg_setup builds from a copy; K is consumed (a second take fails)."""
    K, _ = amg.iga_poisson(3, 3, 8)
    Kc, _ = amg.iga_poisson(3, 3, 8, keep_c=True)
    assert isinstance(Kc, amg.LibCsr) and Kc.nnz == K.nnz
    assert np.array_equal(Kc.to_scipy().data.view(np.uint64), K.to_scipy().data.view(np.uint64))
    H = amg.Hierarchy(K, amg.params(3, host_only=1))
    Ht = amg.Hierarchy(Kc, amg.params(3, host_only=1), take=True)
    with pytest.raises(ValueError):
        Kc.take()
    assert Kc.shape == K.shape
    for l in range(H.info()["levels"]):
        a, b = H.export(l), Ht.export(l)
        assert _bitwise(a["K"].to_scipy(), b["K"].to_scipy())
        if a["P"] is not None:
            assert _bitwise(a["P"].to_scipy(), b["P"].to_scipy())
    # the symmetry check without a transposed copy still rejects a non-symmetric K (one value flipped)
    Kn, _ = amg.iga_poisson(2, 2, 4, keep_c=True)
    Kn.data[1] = Kn.data[1] * 0.5
    with pytest.raises(amg.AmgError, match="symmetric"):
        amg.Hierarchy(Kn, amg.params(2, host_only=1), take=True)


def test_lean_two_pass_setup_bitwise():
    """The two-pass row assembly of the largest levels (AMG_SETUP_LEAN=1: count, then fill the exact
    output; automatic from 8 M rows) builds bitwise the single-pass hierarchy."""
    import hashlib
    import subprocess
    import sys
    code = (
        "import sys, hashlib, numpy as np; sys.path.insert(0, %r)\n"
        "import paper_2511_21268_b200 as amg\n"
        "K, _ = amg.iga_poisson(3, 2, 14)\n"
        "H = amg.Hierarchy(K, amg.params(2, host_only=1))\n"
        "h = hashlib.sha256()\n"
        "for l in range(H.info()['levels']):\n"
        "    e = H.export(l)\n"
        "    for M in (e['K'], e['P']):\n"
        "        if M is not None:\n"
        "            for a in (M.indptr, M.indices, M.data): h.update(np.ascontiguousarray(a).tobytes())\n"
        "print(h.hexdigest())\n") % ROOT
    out = {}
    for lean in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                           env=dict(os.environ, AMG_SETUP_LEAN=lean), timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[lean] = r.stdout.strip().splitlines()[-1]
    assert out["0"] == out["1"]


def test_solve_without_device_part_fails_loudly():
    K, F = amg.iga_poisson(2, 2, 4)
    H = amg.Hierarchy(K.to_scipy(), amg.params(2, host_only=1))
    with pytest.raises(amg.AmgError, match="ENODEV"):
        H.solve_host(F)


@pytest.mark.parametrize("p,n", [(1, 7), (2, 16), (3, 12), (4, 9), (5, 11), (6, 20)])
def test_tables_bitwise_equal_exact_rationals(p, n):
    """c.3: binary128 Gauss + one rounding == correctly rounded exact rationals, every entry."""
    M, K = amg.iga_tables(p, n)
    Mo, Ko = tables.hat_tables(p, n)
    assert np.array_equal(M, Mo) and np.array_equal(K, Ko)


def _bitwise(a, b):
    return (a.shape == b.shape and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
            and np.array_equal(a.data.view(np.uint64), b.data.view(np.uint64)))


@pytest.mark.parametrize("dim,p,n,sides", [(2, 2, 16, 7), (3, 2, 8, 7), (3, 3, 12, 7), (3, 4, 6, 7),
                                           (3, 2, 5, 0), (3, 3, 4, 0b111111), (2, 1, 9, 0b1010)])
def test_generator_bitwise(dim, p, n, sides):
    """c.4: the library's K is bitwise the oracle's; the load vectors agree to 1e-14 (c.5)."""
    K, F = amg.iga_poisson(dim, p, n, sides)
    Ko = oracle.assemble(dim, p, n, sides)
    assert _bitwise(K.to_scipy(), Ko)
    if sides == 7:
        from oracle import bspline
        Fo = bspline.load_vector(dim, p, n, sides)
        assert np.abs(F - Fo).max() <= 1e-14 * np.abs(Fo).max()


def _compare_hierarchies(H, Ho):
    info = H.info()
    assert info["N"] == [L.N for L in Ho.levels]
    for l, Lo in enumerate(Ho.levels):
        e = H.export(l)
        assert _bitwise(e["K"].to_scipy(), Lo.K), f"K_{l}"
        assert np.array_equal(e["dhat"], Lo.dhat), f"dhat_{l}"
        if Lo.P is None:
            assert e["P"] is None and e["agg"] is None
        else:
            assert np.array_equal(e["agg"], Lo.agg), f"aggregates_{l}"
            assert _bitwise(e["P"].to_scipy(), Lo.P), f"P_{l}"
            assert e["omega"] == Lo.omega
    assert info["opc"] == pytest.approx(Ho.opc(), rel=1e-15)


@pytest.mark.parametrize("dim,p,n,kw", [
    (2, 2, 16, {}),                                  # C1
    (3, 3, 12, {}),
    (3, 2, 32, {}),                                  # C2
    (3, 4, 10, {}),
    (3, 3, 12, dict(filter_theta=0.0)),              # literal (I − ωD⁻¹K)P
    (3, 2, 10, dict(smooth_prolong=0)),              # unsmoothed
    (3, 2, 10, dict(agg_steps=1, coarse_size=20)),   # pairwise aggregation, deeper hierarchy
    (3, 3, 8, dict(match_threshold=0.0)),            # maximal matching eligibility
])
def test_setup_bitwise_vs_oracle(dim, p, n, kw):
    """c.6-c.15: aggregate maps, patterns AND values of every level bitwise equal to the oracle."""
    K, _ = amg.iga_poisson(dim, p, n)
    prm = amg.params(p, host_only=1, **kw)
    H = amg.Hierarchy(K, prm)
    okw = {k: v for k, v in kw.items()}
    Ho = oracle.setup(oracle.assemble(dim, p, n), oracle.OParams.for_degree(p, **okw))
    _compare_hierarchies(H, Ho)


@pytest.mark.parametrize("threads", [1, 3])
def test_setup_independent_of_thread_count(threads):
    K, _ = amg.iga_poisson(3, 2, 12)
    ref = amg.Hierarchy(K, amg.params(2, host_only=1))
    H = amg.Hierarchy(K, amg.params(2, host_only=1, num_threads=threads))
    for l in range(ref.info()["levels"]):
        a, b = ref.export(l), H.export(l)
        assert _bitwise(a["K"].to_scipy(), b["K"].to_scipy())


@pytest.mark.parametrize("p,n", [(2, 3), (3, 4), (3, 12), (5, 6), (6, 6)])
def test_paper_cube_load_matches_oracle(p, n):
    """rhs = 2 (the paper's own cube data): library F (binary128 moments, CG boundary
    projection) vs the oracle's separable route (fp64 moments, sparse direct projection)."""
    from oracle import cube_paper
    K, F = amg.iga_poisson(3, p, n, rhs=2)
    Fo, _ = cube_paper.paper_cube_rhs(p, n)
    assert np.abs(F - Fo).max() <= 1e-13 * np.abs(Fo).max()


def test_paper_cube_load_rejects_other_geometries():
    with pytest.raises(amg.AmgError):
        amg.iga_poisson(2, 2, 8, rhs=2)


def test_no_undefined_internal_symbols():
    """Every kernel launcher the runtime uses is instantiated in the library (a missing explicit
    instantiation would only fail at load time on the GPU box)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--undefined-only", _lib.LIB_PATH if hasattr(_lib, "LIB_PATH") else
                          os.path.join(ROOT, "paper_2511_21268_b200", "libamg_b200.so")],
                         capture_output=True, text=True).stdout
    assert "amgb" not in out


@pytest.mark.parametrize("p,n", [(2, 3), (3, 6), (4, 5)])
def test_ring_operator_bitwise_equal_to_oracle(p, n):
    """geometry = 1 (thick quarter ring, NEXT-3): correctly rounded weighted 1-D tables on both sides
    and the canonical evaluation order make K bitwise equal."""
    from oracle import ring
    K, F = amg.iga_poisson(3, p, n, rhs=1, geometry=1)
    Ko = ring.assemble_ring(p, n)
    assert np.array_equal(K.indptr, Ko.indptr) and np.array_equal(K.indices, Ko.indices)
    assert np.array_equal(K.data.view(np.uint64), Ko.data.view(np.uint64))
    assert not F.any()


def test_ring_hierarchy_bitwise_equal_to_oracle():
    from oracle import ring
    p, n = 3, 8
    K, _ = amg.iga_poisson(3, p, n, rhs=1, geometry=1)
    H = amg.Hierarchy(K, amg.params(p, host_only=1))
    Ho = oracle.setup(ring.assemble_ring(p, n), oracle.OParams.for_degree(p))
    assert H.info()["levels"] == Ho.nlevels
    for l, L in enumerate(Ho.levels):
        e = H.export(l)
        Kl = e["K"]
        assert np.array_equal(Kl.indices, L.K.indices) and np.array_equal(Kl.data.view(np.uint64), L.K.data.view(np.uint64))
        if L.P is not None:
            assert np.array_equal(e["P"].data.view(np.uint64), L.P.data.view(np.uint64))


def test_ring_rejects_bad_combinations():
    with pytest.raises(amg.AmgError):
        amg.iga_poisson(2, 2, 4, rhs=1, geometry=1)
    with pytest.raises(amg.AmgError):
        amg.iga_poisson(3, 2, 4, rhs=0, geometry=1)  # the manufactured sine is a cube solution


@pytest.mark.parametrize("p,n", [(2, 3), (3, 6), (4, 5)])
def test_paper_ring_load_matches_oracle(p, n):
    from oracle import ring
    K, F = amg.iga_poisson(3, p, n, rhs=2, geometry=1)
    Fo, _ = ring.paper_ring_rhs(p, n)
    assert np.abs(F - Fo).max() <= 1e-13 * np.abs(Fo).max()


@pytest.mark.parametrize("p,n", [(1, 3), (2, 3), (3, 4), (4, 2)])
def test_lshape_operator_bitwise_equal_to_oracle(p, n):
    """geometry = 2 (three-patch L-shape, NEXT-4): patch entries summed in patch order on both sides,
    so K is bitwise the oracle's glued Σ_P S_Pᵀ K_cube S_P restricted to the free DOFs; the f = 1 load
    (rhs = 0) agrees with the oracle's quadrature to 1e-13."""
    from oracle import lshape
    K, F = amg.iga_poisson(3, p, n, rhs=0, geometry=2)
    Ko = lshape.assemble_lshape(p, n)
    assert np.array_equal(K.indptr, Ko.indptr) and np.array_equal(K.indices, Ko.indices)
    assert np.array_equal(K.data.view(np.uint64), Ko.data.view(np.uint64))
    free, _, _ = lshape.free_lists(p, n)
    zero = lambda x, y, z: 0.0 * x  # noqa: E731
    Fo = lshape.load_all(p, n, f=lambda x, y, z: 1.0 + 0.0 * x, gN4=zero, gN6=zero)[free]
    assert np.abs(F - Fo).max() <= 1e-13 * np.abs(Fo).max()
    assert not amg.iga_poisson(3, p, n, rhs=1, geometry=2)[1].any()


def test_lshape_sizes_table2b():
    """Library sizes at k = 12 against Table 2b (p = 5 is the table's misprint 11,024 → 11,040)."""
    for p, size in [(2, 5772), (3, 7280), (4, 9030), (5, 11040), (6, 13328)]:
        assert amg.iga_poisson(3, p, 12, rhs=1, geometry=2)[0].shape[0] == size


def test_lshape_hierarchy_bitwise_equal_to_oracle():
    from oracle import lshape
    p, n = 3, 6
    K, _ = amg.iga_poisson(3, p, n, rhs=1, geometry=2)
    H = amg.Hierarchy(K, amg.params(p, host_only=1))
    Ho = oracle.setup(lshape.assemble_lshape(p, n), oracle.OParams.for_degree(p))
    assert H.info()["levels"] == Ho.nlevels
    for l, L in enumerate(Ho.levels):
        e = H.export(l)
        assert np.array_equal(e["K"].indices, L.K.indices)
        assert np.array_equal(e["K"].data.view(np.uint64), L.K.data.view(np.uint64))
        if L.P is not None:
            assert np.array_equal(e["agg"], L.agg)
            assert np.array_equal(e["P"].data.view(np.uint64), L.P.data.view(np.uint64))


def test_lshape_rejects_bad_combinations():
    with pytest.raises(amg.AmgError):
        amg.iga_poisson(2, 2, 4, rhs=1, geometry=2)
    with pytest.raises(amg.AmgError):
        amg.iga_poisson(3, 2, 4, dirichlet_sides=0, rhs=1, geometry=2)
    with pytest.raises(amg.AmgError):
        amg.iga_poisson(3, 2, 4, rhs=1, geometry=3)


@pytest.mark.parametrize("p,n", [(1, 3), (2, 3), (3, 4), (4, 2)])
def test_paper_lshape_load_matches_oracle(p, n):
    """rhs = 2 on the L-shape: the library's source, Neumann faces, joint Dirichlet projection (its own
    Jacobi-CG) and lifting agree with the oracle's (sparse direct projection) to 1e-13."""
    from oracle import lshape
    _, F = amg.iga_poisson(3, p, n, rhs=2, geometry=2)
    Fo, _ = lshape.paper_lshape_rhs(p, n)
    assert np.abs(F - Fo).max() <= 1e-13 * np.abs(Fo).max()
