"""GPU parity of the CUDA solve path against the oracle (element by element), through the C ABI.

Tolerances: device sums run in a different order than the oracle's sequential ones and
use FMA, so operator applications agree to a few ulps of Σ|a_ij x_j| (checked at 1e-13 relative to
that bound), one V-cycle to 1e-12 relative (max-norm), the PCG solution after the same number of
iterations to 1e-10 relative, and PCG iteration counts at rtol 1e-6 within ±1 (north star).
"""
import os

import numpy as np
import pytest

import oracle
from oracle import bspline
import amg_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _amg():
    import paper_2511_21268_b200 as amg
    return amg


CASES = {
    "C1": (2, 2, 16),
    "cube12p3": (3, 3, 12),
    "C2": (3, 2, 32),
    "cube10p4": (3, 4, 10),
}

_cache = {}


# 0 the bench default (the fixed SELL-VI rule for the large K_l / P̄_l, autotuned CSR elsewhere: C2's
# K_0 and P̄_0 are SELL-VI), 1 CSR2 (warp per row group), 2 SELL2 (row per lane), 3 CSR4T (TMA-staged
# rows), 4 CSR2 with 16-bit column offsets, 5 CSR4T with 16-bit column offsets, 6 SELL-VI wherever
# admissible
FORMATS = [0, 1, 2, 3, 4, 5, 6]


def build(case, fmt=0, **kw):
    key = (case, fmt, tuple(sorted(kw.items())))
    if key not in _cache:
        amg = _amg()
        dim, p, n = CASES[case]
        K, F = amg.iga_poisson(dim, p, n)
        H = amg.Hierarchy(K, amg.params(p, format=fmt, **kw))
        Ho = oracle.setup(K.to_scipy(), oracle.OParams.for_degree(p, **kw))
        _cache[key] = (K.to_scipy(), F, H, Ho)
    return _cache[key]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("case", list(CASES))
def test_level_operators(case, fmt):
    """K_l, P̄_l and R_l applied on the device vs the oracle's sequential SpMV, every level."""
    K, F, H, Ho = build(case, fmt)
    rng = np.random.default_rng(1)
    for l, L in enumerate(Ho.levels):
        ops = [(0, L.K)] + ([] if L.P is None else [(1, L.P), (2, L.R)])
        for op, A in ops:
            x = rng.uniform(-1, 1, A.shape[1])
            y = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
            H.apply(l, op, dev(x), y)
            ref = oracle.spmv(A, x)
            bound = abs(A) @ np.abs(x)
            assert np.all(np.abs(y.cpu().numpy() - ref) <= 1e-13 * bound + 1e-300), (l, op)


@pytest.mark.parametrize("case", ["C2", "cube10p4"])
def test_kernel_configs_bitwise_equal(case):
    """Every CSR kernel configuration (register / TMA core, int32 / 16-bit-offset columns, rows per warp
    group G, pairs in flight U) sums each row in the same order: y = A·x must be BITWISE identical
    across all of them, and within 1e-13 of the oracle (so the autotuner changes speed, never results)."""
    K, F, H, Ho = build(case, 0)
    rng = np.random.default_rng(5)
    for l, L in enumerate(Ho.levels):
        ops = [(0, L.K)] + ([] if L.P is None else [(1, L.P), (2, L.R)])
        for op, A in ops:
            keep = H.op_config(l, op)
            x = dev(rng.uniform(-1, 1, A.shape[1]))
            ref = None
            if keep["layout"] in ("sellvi", "sellviw"):  # SELL-VI: every U (and window count) sums alike
                ys = []
                for kb in ([1, 2] if keep["layout"] == "sellviw" else [0]):
                    for U in (1, 2, 4):
                        H.set_op_config(l, op, kb, 32, U)
                        y = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
                        H.apply(l, op, x, y)
                        ys.append(y.cpu().numpy())
                xo = x.cpu().numpy()
                assert np.all(np.abs(ys[0] - oracle.spmv(A, xo)) <= 1e-13 * (abs(A) @ np.abs(xo)) + 1e-300)
                assert all(np.array_equal(y, ys[0]) for y in ys)
                H.set_op_config(l, op, keep["kernel_bits"], 32, keep["U"])
                continue
            kerns = [0, 1, 2, 3, 4, 6]  # bit 0 TMA, bit 1 16-bit columns, bit 2 L2 prefetch
            if keep["n_values"]:  # bit 3: value index (CSR-VI), register core
                kerns += [8, 10, 12, 14]
            for kern in kerns:
                for G in (1, 2, 4, 8, 32):
                    for U in (2, 4, 6, 8):
                        if (kern & 1) and U > 4:
                            continue
                        H.set_op_config(l, op, kern, G, U)
                        y = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
                        H.apply(l, op, x, y)
                        y = y.cpu().numpy()
                        if ref is None:
                            ref = y
                            xo = x.cpu().numpy()
                            bound = abs(A) @ np.abs(xo)
                            assert np.all(np.abs(y - oracle.spmv(A, xo)) <= 1e-13 * bound + 1e-300)
                        else:
                            assert np.array_equal(y, ref), (l, op, kern, G, U)
            H.set_op_config(l, op, keep["kernel_bits"], keep["G"], keep["U"])


def test_d16_encoding_bytes():
    """16-bit column offsets: the fine IgA operator qualifies (every row spans < 65536 columns) and
    the reported algorithmic bytes follow the chosen column source exactly."""
    K, F, H, Ho = build("cube12p3", 0)
    c = H.op_config(0, 0)
    H.set_op_config(0, 0, 2, c["G"], c["U"])
    d16 = H.op_config(0, 0)
    H.set_op_config(0, 0, 0, c["G"], c["U"])
    i32 = H.op_config(0, 0)["alg_bytes"]
    H.set_op_config(0, 0, c["kernel_bits"], c["G"], c["U"])
    nnz, N = c["nnz"], K.shape[0]
    assert i32 == 12 * nnz + 8 * (N + 1)
    assert d16["alg_bytes"] == 10 * nnz + 4 * N + 8 * (N + 1)


@pytest.mark.parametrize("windowed", [0, 1])
def test_sellvi_layout(windowed, monkeypatch):
    """SELL-VI (format 6; format 0 picks it for the large K_l): row per lane, one 32-bit word per entry
    (16-bit column offset | 16-bit value index; windowed: window position | value index).  The table
    holds exactly the distinct values (+0.0 of the padding), the reported bytes are 4 B per non-zero +
    the table + row bases + slice offsets (windowed: no row bases; + 16 B per block and per window run),
    every U (and window count) gives bitwise the same y, and y matches the oracle's SpMV on every level's
    K_l, P̄_l and R_l."""
    monkeypatch.setenv("AMG_SELLVI_WIN", str(windowed))
    amg = _amg()
    dim, p, n = CASES["C2"]
    K, F = amg.iga_poisson(dim, p, n)
    H = amg.Hierarchy(K, amg.params(p, format=6))
    Ho = build("C2", 6)[3]
    layout = "sellviw" if windowed else "sellvi"
    rng = np.random.default_rng(11)
    seen = 0
    for l, L in enumerate(Ho.levels):
        ops = [(0, L.K)] + ([] if L.P is None else [(1, L.P), (2, L.R)])
        for op, A in ops:
            c = H.op_config(l, op)
            if c["layout"] not in ("sellvi", "sellviw"):
                continue
            if op == 0 and l == 0:
                assert c["layout"] == layout, (l, op, c)  # K_0 (159 values, table in shared memory) is windowed
            if c["layout"] == "sellviw":
                assert c["n_values"] <= 8192  # windows only with the value table in shared memory
            seen += 1
            A = A.tocsr()
            bits = np.unique(np.concatenate([A.data.view(np.uint64), np.zeros(1, np.uint64)]))
            assert c["n_values"] == bits.size
            nr = A.shape[0]
            nsl = (nr + 31) // 32
            if c["layout"] == "sellvi":
                assert c["alg_bytes"] == 4 * A.nnz + 8 * bits.size + 4 * nr + 8 * (nsl + 1)
            else:
                base = 4 * A.nnz + 8 * bits.size + 8 * (nsl + 1) + 16 * ((nsl + 7) // 8)
                runs = (c["alg_bytes"] - base) / 16  # 16 B per window run, at least one per block
                assert runs == int(runs) and (nsl + 7) // 8 <= runs <= 32 * nsl
            x = dev(rng.uniform(-1, 1, A.shape[1]))
            ys = []
            for kb in ([1, 2] if c["layout"] == "sellviw" else [0]):
                for U in (1, 2, 4):
                    H.set_op_config(l, op, kb, 32, U)
                    y = torch.empty(nr, dtype=torch.float64, device="cuda")
                    H.apply(l, op, x, y)
                    ys.append(y.cpu().numpy())
            H.set_op_config(l, op, c["kernel_bits"], 32, c["U"])
            xo = x.cpu().numpy()
            assert all(np.array_equal(y, ys[0]) for y in ys)
            assert np.all(np.abs(ys[0] - oracle.spmv(A, xo)) <= 1e-13 * (abs(A) @ np.abs(xo)) + 1e-300)
    assert seen >= 1  # at least C2's K_0 (159 distinct values) qualifies


def test_sellvi_windowed_bitwise_equals_plain(monkeypatch):
    """The windowed core (x staged in shared memory, window positions in the words) sums every row in
    the plain SELL-VI order: y = A·x on every level and one V-cycle are BITWISE those of the plain
    layout (AMG_SELLVI_WIN=0), for the bench's format 0 and for format 6, also with the windowed tail
    items forced to single slices (AMG_SELLVIW_SPLIT=3: slices stay whole).  (The plain layout's tail
    split — on at C2's few slices per warp — sums a row's parts separately, so it is switched off:
    AMG_SELLVI_PARTS=0; the split against the unsplit sum is test_sellvi_split_slices.)"""
    amg = _amg()
    dim, p, n = CASES["C2"]
    monkeypatch.setenv("AMG_SELLVI_PARTS", "0")
    for fmt, split in ((0, None), (6, None), (0, "3")):
        Hs = {}
        for wnd in (0, 1):
            monkeypatch.setenv("AMG_SELLVI_WIN", str(wnd))
            if split is not None and wnd == 1:  # windowed tail items of 1 slice for every block
                monkeypatch.setenv("AMG_SELLVIW_SPLIT", split)
            K, F = amg.iga_poisson(dim, p, n)
            Hs[wnd] = amg.Hierarchy(K, amg.params(p, format=fmt))
            monkeypatch.delenv("AMG_SELLVIW_SPLIT", raising=False)
        assert Hs[1].op_config(0, 0)["layout"] == "sellviw" and Hs[0].op_config(0, 0)["layout"] == "sellvi"
        info = Hs[0].info()
        rng = np.random.default_rng(31)
        for l in range(info["levels"]):
            for op in ((0, 1, 2) if l + 1 < info["levels"] else (0,)):
                nr = info["N"][l] if op < 2 else info["N"][l + 1]
                ncol = info["N"][l] if op != 1 else info["N"][l + 1]
                x = dev(rng.uniform(-1, 1, ncol))
                ys = []
                for wnd in (0, 1):
                    y = torch.empty(nr, dtype=torch.float64, device="cuda")
                    Hs[wnd].apply(l, op, x, y)
                    ys.append(y.cpu().numpy())
                assert np.array_equal(ys[0], ys[1]), (fmt, l, op)
        r = dev(amg_inputs.uniform_pm1(info["N"][0], seed=41))
        assert torch.equal(Hs[0].vcycle(r), Hs[1].vcycle(r)), fmt


def test_sellvi_wide_offsets():
    """SELL-VI words with more than 16 offset bits (rows spanning > 65535 columns, as at C4 and C5):
    the 7-point Laplacian of a 200 x 200 x 4 grid (couplings at distance 40000, rows spanning 80000
    columns: obits = 17, 15-bit value index) applied through the SELL-VI core matches scipy's product."""
    amg = _amg()
    import scipy.sparse as sp

    def lap1(m):
        return sp.diags([2.0 * np.ones(m), -np.ones(m - 1), -np.ones(m - 1)], [0, -1, 1])

    nx, ny, nz = 200, 200, 4
    Ix, Iy, Iz = sp.identity(nx), sp.identity(ny), sp.identity(nz)
    A = (sp.kron(sp.kron(Iz, Iy), lap1(nx)) + sp.kron(sp.kron(Iz, lap1(ny)), Ix)
         + sp.kron(sp.kron(lap1(nz), Iy), Ix)).tocsr()
    A.sort_indices()
    n = A.shape[0]
    H = amg.Hierarchy(A, amg.params(2, format=6))
    c = H.op_config(0, 0)
    assert c["layout"] == "sellviw"  # the windows (3 runs of ~650 columns per block) make the width moot
    os.environ["AMG_SELLVI_WIN"] = "0"
    try:
        H0 = amg.Hierarchy(A, amg.params(2, format=6))
    finally:
        del os.environ["AMG_SELLVI_WIN"]
    c = H0.op_config(0, 0)
    assert c["layout"] == "sellvi" and c["offset_bits"] == 17
    x = np.random.default_rng(4).uniform(-1, 1, n)
    for Hh in (H, H0):
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        Hh.apply(0, 0, dev(x), y)
        assert np.allclose(y.cpu().numpy(), A @ x, rtol=0, atol=1e-13 * 12)


@pytest.mark.parametrize("lparts", [1, 2, 3])
def test_sellvi_split_slices(lparts, monkeypatch):
    """SELL-VI slices split into 2^lparts quad ranges, one warp each (the tail round's setting, forced
    on every slice here by AMG_SELLVI_PARTS): K_0 of C2 matches the oracle's SpMV, the solve converges in the
    unsplit solve's iterations to the same solution (only the order of the two partial sums per part
    changes), and U does not change the bits."""
    amg = _amg()
    K, F, H0, Ho = build("C2", 6)
    monkeypatch.setenv("AMG_SELLVI_PARTS", str(lparts))
    monkeypatch.setenv("AMG_SELLVI_WIN", "0")  # the split is a feature of the plain (multi-GPU) layout
    H = amg.Hierarchy(amg.iga_poisson(*CASES["C2"])[0], amg.params(CASES["C2"][1], format=6))
    c = H.op_config(0, 0)
    assert c["layout"] == "sellvi" and c["sellvi_parts"] == 1 << lparts
    A = Ho.levels[0].K.tocsr()
    x = dev(np.random.default_rng(12).uniform(-1, 1, A.shape[0]))
    ys = []
    for U in (1, 2, 4):
        H.set_op_config(0, 0, 0, 32, U)
        y = torch.empty(A.shape[0], dtype=torch.float64, device="cuda")
        H.apply(0, 0, x, y)
        ys.append(y.cpu().numpy())
    xo = x.cpu().numpy()
    assert all(np.array_equal(y, ys[0]) for y in ys)
    assert np.all(np.abs(ys[0] - oracle.spmv(A, xo)) <= 1e-13 * (abs(A) @ np.abs(xo)) + 1e-300)
    Fd = dev(F)
    u0, it0 = H0.solve(Fd, rtol=1e-8, maxit=200)[:2]
    u1, it1 = H.solve(Fd, rtol=1e-8, maxit=200)[:2]
    assert it1 == it0
    u0, u1 = u0.cpu().numpy(), u1.cpu().numpy()
    assert np.linalg.norm(u1 - u0) <= 1e-10 * np.linalg.norm(u0)


def test_value_index_table():
    """CSR-VI (kernel bit 3): the value table of C2's K_0 holds exactly the distinct stored values
    (the operator's values and the 0.0 of the row padding, counted here by numpy on the host K), the
    reported bytes follow the packed 4 B/entry format, and y = K_0 x through the value-indexed cores
    is bitwise the streamed-value result and within 1e-13 of the oracle."""
    K, F, H, Ho = build("C2", 4)  # CSR layout everywhere (format 0 would store C2's K_0 as SELL-VI)
    c = H.op_config(0, 0)
    bits = np.unique(np.concatenate([K.data.view(np.uint64), np.zeros(1, np.uint64)]))
    assert c["n_values"] == bits.size and c["value_index_bytes"] == 2
    N, nnz = K.shape[0], K.nnz
    x = dev(np.random.default_rng(9).uniform(-1, 1, N))
    ys = {}
    for kern in (2, 10, 14, 8, 12):
        H.set_op_config(0, 0, kern, c["G"], c["U"])
        y = torch.empty(N, dtype=torch.float64, device="cuda")
        H.apply(0, 0, x, y)
        ys[kern] = y.cpu().numpy()
        if kern == 10:
            assert H.op_config(0, 0)["alg_bytes"] == 4 * nnz + 4 * N + 8 * bits.size + 8 * (N + 1)
        if kern == 8:  # int32 columns + 32-bit value index
            assert H.op_config(0, 0)["alg_bytes"] == 8 * nnz + 8 * bits.size + 8 * (N + 1)
    H.set_op_config(0, 0, c["kernel_bits"], c["G"], c["U"])
    for kern, y in ys.items():
        assert np.array_equal(y, ys[2]), kern
    xo = x.cpu().numpy()
    assert np.all(np.abs(ys[10] - oracle.spmv(Ho.levels[0].K, xo)) <= 1e-13 * (abs(Ho.levels[0].K) @ np.abs(xo)))


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("case", list(CASES))
def test_vcycle(case, fmt):
    """One V-cycle (c.18: Chebyshev pre/post smoothing, restriction, coarse solve, prolongation)."""
    K, F, H, Ho = build(case, fmt)
    for seed in (3, 4):
        r = amg_inputs.uniform_pm1(K.shape[0], seed=seed)
        z = H.vcycle(dev(r)).cpu().numpy()
        zo = oracle.vcycle(Ho, r)
        assert np.abs(z - zo).max() <= 1e-12 * np.abs(zo).max()


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("case", list(CASES))
def test_pcg_fixed_iterations_and_counts(case, fmt):
    """c.19: same iterate after the same number of iterations (1e-10), and iteration counts at
    rtol 1e-6 equal within ±1, for the manufactured RHS and a seeded random RHS."""
    K, F, H, Ho = build(case, fmt)
    for rhs in (F, amg_inputs.uniform_pm1(K.shape[0])):
        uo, ito, rro, histo, rco = oracle.pcg(Ho, rhs, rtol=1e-6, maxit=200)
        assert rco == 0
        u, it, rr, hist, st = H.solve(dev(rhs), rtol=1e-6, maxit=200)
        assert st == 0 and abs(it - ito) <= 1
        assert rr <= 1e-6
        u2, it2, _, hist2, _ = H.solve(dev(rhs), rtol=0.0, maxit=ito)
        assert it2 == ito
        uo_n = np.linalg.norm(uo)
        assert np.linalg.norm(u2.cpu().numpy() - uo) <= 1e-10 * uo_n
        assert np.allclose(hist2, histo, rtol=1e-8, atol=0)
        # true residual of the converged device solution
        ud = u.cpu().numpy()
        assert np.linalg.norm(rhs - oracle.spmv(K, ud)) <= 1.05e-6 * np.linalg.norm(rhs)


def test_host_pointer_entry_matches_device_entry():
    K, F, H, Ho = build("C2")
    u_dev, it, rr, _, _ = H.solve(dev(F))
    u_host, it2, rr2, _ = H.solve_host(F)
    assert it == it2 and np.array_equal(u_dev.cpu().numpy(), u_host)


@pytest.mark.parametrize("krylov", [0, 1])
def test_device_loop_equals_host_loop(krylov, monkeypatch):
    """The Krylov loop on the device (one graph with a conditional WHILE node, k_loop_ctl deciding) gives
    BITWISE the iterate, the iteration count, the status and the residual history of the per-iteration
    graphs with the host's stopping test (AMG_DEVICE_LOOP=0): converged, cut at maxit, rtol = 0, and a
    zero right-hand side; PCG and FCG with the §5.1 coarse CG."""
    amg = _amg()
    dim, p, n = CASES["C2"]
    Hs = {}
    for dl in (0, 1):
        monkeypatch.setenv("AMG_DEVICE_LOOP", str(dl))
        K, F = amg.iga_poisson(dim, p, n, rhs=2 if krylov else 0)
        Hs[dl] = amg.Hierarchy(K, amg.params(p, krylov=krylov, coarse_solver=krylov))
    Fd = dev(F)
    for rtol, maxit, rhs in ((1e-8, 200, Fd), (1e-8, 3, Fd), (0.0, 5, Fd), (1e-6, 50, torch.zeros_like(Fd))):
        out = []
        for dl in (0, 1):
            u, it, rr, hist, st = Hs[dl].solve(rhs, rtol=rtol, maxit=maxit)
            out.append((u.cpu().numpy(), it, rr, np.asarray(hist), st))
        (u0, i0, r0, h0, s0), (u1, i1, r1, h1, s1) = out
        assert (i0, s0) == (i1, s1) and np.array_equal(u0, u1), (rtol, maxit, i0, i1, s0, s1)
        assert r0 == r1 and np.array_equal(h0, h1, equal_nan=True)


def test_deterministic_runs():
    K, F, H, Ho = build("cube12p3")
    a = H.solve(dev(F))[0].cpu().numpy()
    b = H.solve(dev(F))[0].cpu().numpy()
    assert np.array_equal(a, b)


def test_edge_cases():
    amg = _amg()
    K, F, H, Ho = build("C1")
    # F = 0 -> u = 0, 0 iterations
    u, it, rr, hist, st = H.solve(torch.zeros(K.shape[0], dtype=torch.float64, device="cuda"))
    assert it == 0 and st == 0 and not u.any()
    # maxit = 0 -> not converged, u unchanged (0)
    u, it, rr, hist, st = H.solve(dev(F), maxit=0)
    assert it == 0 and st == 1 and not u.any()
    # nonzero initial guess: start from the exact-ish solution -> converges immediately
    uo = oracle.pcg(Ho, F, rtol=1e-12)[0]
    u, it, rr, hist, st = H.solve(dev(F), u=dev(uo), rtol=1e-6)
    assert it == 0 and st == 0
    # single-level hierarchy (N <= coarse_size): V = 30 ℓ1-Jacobi sweeps
    Ks, Fs = amg.iga_poisson(2, 2, 4)
    Hs = amg.Hierarchy(Ks, amg.params(2, coarse_size=1000))
    Hso = oracle.setup(Ks.to_scipy(), oracle.OParams.for_degree(2, coarse_size=1000))
    assert Hs.info()["levels"] == 1
    r = amg_inputs.uniform_pm1(Ks.shape[0], seed=7)
    assert np.abs(Hs.vcycle(dev(r)).cpu().numpy() - oracle.vcycle(Hso, r)).max() <= 1e-12 * np.abs(r).max()
    # degree-1 smoother and odd degree paths
    for m, fmt in ((1, 1), (3, 2), (2, 2)):
        Km, Fm = amg.iga_poisson(3, 2, 8)
        Hm = amg.Hierarchy(Km, amg.params(2, cheb_degree=m, format=fmt))
        Hmo = oracle.setup(Km.to_scipy(), oracle.OParams(cheb_degree=m))
        r = amg_inputs.uniform_pm1(Km.shape[0], seed=8)
        zo = oracle.vcycle(Hmo, r)
        assert np.abs(Hm.vcycle(dev(r)).cpu().numpy() - zo).max() <= 1e-12 * np.abs(zo).max()


@pytest.mark.parametrize("fmt", [0, 1])
def test_c3_full_size_properties(fmt):
    """C3 (k=96, p=3; 941,094 DOFs) in the bench's configuration: hierarchy identical to the host
    export, level-0 SpMV vs the oracle on all rows, V-cycle symmetry, converged true residual."""
    amg = _amg()
    K, F = amg.iga_poisson(3, 3, 96)
    Ks = K.to_scipy()
    H = amg.Hierarchy(K, amg.params(3, format=fmt))
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, Ks.shape[0])
    y = torch.empty(Ks.shape[0], dtype=torch.float64, device="cuda")
    H.apply(0, 0, dev(x), y)
    ref = oracle.spmv(Ks, x)
    assert np.all(np.abs(y.cpu().numpy() - ref) <= 1e-13 * (abs(Ks) @ np.abs(x)))
    r1 = dev(amg_inputs.uniform_pm1(Ks.shape[0], seed=1))
    r2 = dev(amg_inputs.uniform_pm1(Ks.shape[0], seed=2))
    a = torch.dot(H.vcycle(r1), r2).item()
    b = torch.dot(r1, H.vcycle(r2)).item()
    assert abs(a - b) <= 1e-11 * abs(a)
    u, it, rr, hist, st = H.solve(dev(F), rtol=1e-6)
    assert st == 0 and 5 <= it <= 40
    ud = u.cpu().numpy()
    assert np.linalg.norm(F - oracle.spmv(Ks, ud)) <= 1.05e-6 * np.linalg.norm(F)


def test_c3_paper_solve_vs_oracle_artifact():
    """The bench's default solve at full size — C3 (k=96, p=3, 941,094 DOFs), the paper's experiment
    (its data, FCG, §5.1 coarse CG), format 0 (SELL-VI K_0 / P̄_0, autotuned CSR elsewhere) — against
    the oracle's own C3 solve committed in oracle/sizes_C3.json (written by the oracle-only script
    oracle/scripts/hierarchy_sizes.py): level sizes and nnz equal, iteration count ±1, the residual
    history of the oracle's iterations to 1e-8 relative, and the iterate after the oracle's iteration
    count on every 997th row to 1e-10 of its max."""
    import json
    import os
    amg = _amg()
    with open(os.path.join(os.path.dirname(oracle.__file__), "sizes_C3.json")) as f:
        art = json.load(f)
    K, F = amg.iga_poisson(3, 3, 96, rhs=2)
    H = amg.Hierarchy(K, amg.params(3, krylov=1, coarse_solver=1))
    info = H.info()
    assert info["N"] == art["N"] and info["nnz"] == art["nnz"]
    Fd = dev(F)
    ito = art["oracle_iters_paper"]
    u, it, rr, hist, st = H.solve(Fd, rtol=1e-6, maxit=200)
    assert st == 0 and abs(it - ito) <= 1, (it, ito)
    u2, it2, _, hist2, _ = H.solve(Fd, rtol=0.0, maxit=ito)
    assert it2 == ito
    assert np.allclose(hist2, art["oracle_hist_paper"], rtol=1e-8, atol=0)
    idx = list(range(0, K.shape[0], art["u_sample_stride"])) + [K.shape[0] - 1]
    us = u2.cpu().numpy()[idx]
    uo = np.array(art["u_sample_paper"])
    assert np.abs(us - uo).max() <= 1e-10 * np.abs(uo).max()


# --- NEXT-1: the paper's own cube experiment --------------------
def test_coarse_cg_vcycle_matches_oracle():
    """§5.1 coarsest solver (CG with one weighted-Jacobi sweep as preconditioner) inside the V-cycle:
    with tolerance 0 and 30 iterations both sides reach the coarse solution to round-off."""
    amg = _amg()
    dim, p, n = CASES["cube12p3"]
    K, F = amg.iga_poisson(dim, p, n)
    H = amg.Hierarchy(K, amg.params(p, coarse_solver=1, coarse_tol=0.0, coarse_maxit=30))
    Ho = oracle.setup(K.to_scipy(), oracle.OParams.for_degree(p, coarse_solver=1, coarse_tol=0.0, coarse_maxit=30))
    for seed in (3, 4):
        r = amg_inputs.uniform_pm1(K.shape[0], seed=seed)
        z = H.vcycle(dev(r)).cpu().numpy()
        zo = oracle.vcycle(Ho, r)
        assert np.abs(z - zo).max() <= 1e-11 * np.abs(zo).max()


@pytest.mark.parametrize("case", ["cube12p3", "cube10p4"])
def test_fcg_matches_oracle(case):
    """Notay FCG(1) outer solver with the linear V-cycle: same iterate after the oracle's iteration
    count (1e-10) and iteration counts within ±1."""
    amg = _amg()
    dim, p, n = CASES[case]
    K, F = amg.iga_poisson(dim, p, n)
    H = amg.Hierarchy(K, amg.params(p, krylov=1))
    Ho = oracle.setup(K.to_scipy(), oracle.OParams.for_degree(p))
    for rhs in (F, amg_inputs.uniform_pm1(K.shape[0])):
        uo, ito, rro, histo, rco = oracle.fcg(Ho, rhs, rtol=1e-6, maxit=200)
        u, it, rr, hist, st = H.solve(dev(rhs), rtol=1e-6, maxit=200)
        assert rco == 0 and st == 0 and abs(it - ito) <= 1
        u2 = H.solve(dev(rhs), rtol=0.0, maxit=ito)[0].cpu().numpy()
        assert np.linalg.norm(u2 - uo) <= 1e-10 * np.linalg.norm(uo)


@pytest.mark.parametrize("p,n", [(3, 12), (4, 8), (5, 6), (6, 6)])
def test_paper_cube_experiment(p, n):
    """The paper's configuration end to end: its data (rhs = 2), FCG outer, §5.1 coarse CG (1e-4 /
    30 its), Chebyshev degree by p.  Iteration counts within ±1 of the oracle's, true
    residual ≤ 1e-6, and the discrete solution within the discretisation error of u = e^{x+z} sin y."""
    from oracle import cube_paper
    amg = _amg()
    K, F = amg.iga_poisson(3, p, n, rhs=2)
    Fo, uD = cube_paper.paper_cube_rhs(p, n)
    H = amg.Hierarchy(K, amg.params(p, krylov=1, coarse_solver=1))
    Ho = oracle.setup(K.to_scipy(), oracle.OParams.for_degree(p, coarse_solver=1))
    uo, ito, rro, histo, rco = oracle.fcg(Ho, F, rtol=1e-6, maxit=200)
    u, it, rr, hist, st = H.solve(dev(F), rtol=1e-6, maxit=200)
    assert rco == 0 and st == 0 and abs(it - ito) <= 1, (it, ito)
    # the iterate after the oracle's iteration count, and the residual history (the §5.1 coarse CG
    # stops on its 1e-4 tolerance: a round-off change of its stop would show far above these bars)
    u2, it2, _, hist2, _ = H.solve(dev(F), rtol=0.0, maxit=ito)
    assert it2 == ito
    assert np.linalg.norm(u2.cpu().numpy() - uo) <= 1e-9 * np.linalg.norm(uo)
    assert np.allclose(hist2, histo, rtol=1e-7, atol=0)
    ud = u.cpu().numpy()
    Ks = K.to_scipy()
    assert np.linalg.norm(F - oracle.spmv(Ks, ud)) <= 1.05e-6 * np.linalg.norm(F)
    err = cube_paper.l2_error_full(p, n, ud, uD)
    exact = cube_paper.l2_error_full(p, n, np.zeros_like(ud), np.zeros_like(uD))  # ‖u‖_L2
    assert err <= 1e-3 * exact


@pytest.mark.parametrize("p,n", [(2, 8), (3, 8)])
def test_ring_solve_matches_oracle(p, n):
    """NEXT-3, the thick quarter ring (non-isoparametric) with a seeded random RHS:
    V-cycle to 1e-12, the PCG iterate after the oracle's iteration count to 1e-10, counts ±1."""
    from oracle import ring
    amg = _amg()
    K, _ = amg.iga_poisson(3, p, n, rhs=1, geometry=1)
    H = amg.Hierarchy(K, amg.params(p))
    Ho = oracle.setup(ring.assemble_ring(p, n), oracle.OParams.for_degree(p))
    r = amg_inputs.uniform_pm1(K.shape[0], seed=31)
    zo = oracle.vcycle(Ho, r)
    assert np.abs(H.vcycle(dev(r)).cpu().numpy() - zo).max() <= 1e-12 * np.abs(zo).max()
    uo, ito, rro, histo, rco = oracle.pcg(Ho, r, rtol=1e-6, maxit=200)
    u, it, rr, hist, st = H.solve(dev(r), rtol=1e-6, maxit=200)
    assert rco == 0 and st == 0 and abs(it - ito) <= 1
    u2 = H.solve(dev(r), rtol=0.0, maxit=ito)[0].cpu().numpy()
    assert np.linalg.norm(u2 - uo) <= 1e-10 * np.linalg.norm(uo)


@pytest.mark.parametrize("p,n", [(2, 8), (3, 8)])
def test_ring_paper_experiment(p, n):
    """The paper's ring configuration: its data (rhs = 2, geometry = 1), FCG, §5.1 coarse CG — counts
    within ±1 of the oracle's and the converged true residual."""
    from oracle import ring
    amg = _amg()
    K, F = amg.iga_poisson(3, p, n, rhs=2, geometry=1)
    H = amg.Hierarchy(K, amg.params(p, krylov=1, coarse_solver=1))
    Ho = oracle.setup(ring.assemble_ring(p, n), oracle.OParams.for_degree(p, coarse_solver=1))
    uo, ito, rro, histo, rco = oracle.fcg(Ho, F, rtol=1e-6, maxit=200)
    u, it, rr, hist, st = H.solve(dev(F), rtol=1e-6, maxit=200)
    assert rco == 0 and st == 0 and abs(it - ito) <= 1, (it, ito)
    # the iterate after the oracle's iteration count, and the residual history (the §5.1 coarse CG
    # stops on its 1e-4 tolerance: a round-off change of its stop would show far above these bars)
    u2, it2, _, hist2, _ = H.solve(dev(F), rtol=0.0, maxit=ito)
    assert it2 == ito
    assert np.linalg.norm(u2.cpu().numpy() - uo) <= 1e-9 * np.linalg.norm(uo)
    assert np.allclose(hist2, histo, rtol=1e-7, atol=0)
    ud = u.cpu().numpy()
    assert np.linalg.norm(F - oracle.spmv(K.to_scipy(), ud)) <= 1.05e-6 * np.linalg.norm(F)


@pytest.mark.parametrize("p,n", [(2, 8), (3, 6)])
def test_lshape_solve_matches_oracle(p, n):
    """NEXT-4, the three-patch L-shape with a seeded random RHS: V-cycle to 1e-12, the
    PCG iterate after the oracle's iteration count to 1e-10, counts ±1."""
    from oracle import lshape
    amg = _amg()
    K, _ = amg.iga_poisson(3, p, n, rhs=1, geometry=2)
    H = amg.Hierarchy(K, amg.params(p))
    Ho = oracle.setup(lshape.assemble_lshape(p, n), oracle.OParams.for_degree(p))
    r = amg_inputs.uniform_pm1(K.shape[0], seed=37)
    zo = oracle.vcycle(Ho, r)
    assert np.abs(H.vcycle(dev(r)).cpu().numpy() - zo).max() <= 1e-12 * np.abs(zo).max()
    uo, ito, rro, histo, rco = oracle.pcg(Ho, r, rtol=1e-6, maxit=200)
    u, it, rr, hist, st = H.solve(dev(r), rtol=1e-6, maxit=200)
    assert rco == 0 and st == 0 and abs(it - ito) <= 1
    u2 = H.solve(dev(r), rtol=0.0, maxit=ito)[0].cpu().numpy()
    assert np.linalg.norm(u2 - uo) <= 1e-10 * np.linalg.norm(uo)


@pytest.mark.parametrize("p,n", [(2, 8), (3, 6)])
def test_lshape_paper_experiment(p, n):
    """The paper's L-shape data (library rhs = 2 vs the oracle's load: source, Neumann faces y=1 on B
    and x=1 on C, joint L2 Dirichlet projection, lifting), FCG with the §5.1 coarse CG: counts ±1 of the oracle, converged
    true residual, and the discrete solution close to u = e^x sin(xy) cos z."""
    from oracle import lshape
    amg = _amg()
    K, F = amg.iga_poisson(3, p, n, rhs=2, geometry=2)
    Fo, uD = lshape.paper_lshape_rhs(p, n)
    assert np.abs(F - Fo).max() <= 1e-13 * np.abs(Fo).max()
    H = amg.Hierarchy(K, amg.params(p, krylov=1, coarse_solver=1))
    Ho = oracle.setup(lshape.assemble_lshape(p, n), oracle.OParams.for_degree(p, coarse_solver=1))
    uo, ito, rro, histo, rco = oracle.fcg(Ho, F, rtol=1e-6, maxit=200)
    u, it, rr, hist, st = H.solve(dev(F), rtol=1e-6, maxit=200)
    assert rco == 0 and st == 0 and abs(it - ito) <= 1, (it, ito)
    # the iterate after the oracle's iteration count, and the residual history (the §5.1 coarse CG
    # stops on its 1e-4 tolerance: a round-off change of its stop would show far above these bars)
    u2, it2, _, hist2, _ = H.solve(dev(F), rtol=0.0, maxit=ito)
    assert it2 == ito
    assert np.linalg.norm(u2.cpu().numpy() - uo) <= 1e-9 * np.linalg.norm(uo)
    assert np.allclose(hist2, histo, rtol=1e-7, atol=0)
    ud = u.cpu().numpy()
    assert np.linalg.norm(F - oracle.spmv(K.to_scipy(), ud)) <= 1.05e-6 * np.linalg.norm(F)
    norm_u = lshape.l2_error_full(p, n, np.zeros_like(ud), np.zeros_like(uD), exact=lshape.exact_u)
    assert lshape.l2_error_full(p, n, ud, uD) <= 1e-3 * norm_u
