"""Exact 1-D B-spline mass/stiffness tables (oracle, c.3 of SURVEY.md §8c).

TEST INFRASTRUCTURE ONLY — see oracle/__init__.py.

Paper passages: PAPER.md P:L69-78 (B-spline basis, open knot vectors, maximal regularity),
P:L551-568 (Galerkin entries k_ij = ∫∇φ_j·∇φ_i, eq:matrix_and_vector_values P:L646-650),
Remark P:L570-573 ((p+1)-point Gauss is exact for these integrands).

The tables are computed on the integer-knot vector (element size h = 1) by EXACT rational
arithmetic: each basis function is built per element by the Cox–de Boor recursion with
``fractions.Fraction`` coefficients, products are integrated exactly, and only the final
value is rounded to the nearest fp64 (``float(Fraction)`` rounds correctly).  The physical
tables on [0,1] with n elements are then M1 = fl(M̂/n), K1 = fl(K̂·n) in fp64.
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache

import numpy as np


def open_knots(p: int, n: int) -> list[int]:
    """Open uniform knot vector on [0, n] with integer interior knots (multiplicity 1 → C^{p-1})."""
    return [0] * (p + 1) + list(range(1, n)) + [n] * (p + 1)


def _pmul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                out[i + j] += x * y
    return out


def _padd(a, b):
    n = max(len(a), len(b))
    return [(a[i] if i < len(a) else 0) + (b[i] if i < len(b) else 0) for i in range(n)]


def _pder(a):
    return [a[k] * k for k in range(1, len(a))] or [Fraction(0)]


def _pint01(a):
    """∫_0^1 Σ a_k ξ^k dξ = Σ a_k/(k+1), exactly."""
    return sum((c / (k + 1) for k, c in enumerate(a)), Fraction(0))


def element_basis(p: int, n: int, e: int):
    """Polynomials (in the local variable ξ = x - e, ξ∈[0,1]) of the p+1 basis functions
    N_{e..e+p} that are non-zero on element [e, e+1]: Cox–de Boor recursion."""
    t = open_knots(p, n)
    s = e + p  # knot span index: t[s] = e, t[s+1] = e+1
    # N_{i,0}: 1 on span s.  Polynomials in ξ; x = ξ + e.
    N = {i: ([Fraction(1)] if i == s else [Fraction(0)]) for i in range(s - p, s + 1)}
    for k in range(1, p + 1):
        newN = {}
        for i in range(s - k, s + 1):
            acc = [Fraction(0)]
            # (x - t_i)/(t_{i+k} - t_i) N_{i,k-1}
            den = t[i + k] - t[i]
            if den != 0 and i in N:
                lin = [Fraction(e - t[i], den), Fraction(1, den)]
                acc = _padd(acc, _pmul(lin, N[i]))
            # (t_{i+k+1} - x)/(t_{i+k+1} - t_{i+1}) N_{i+1,k-1}
            den = t[i + k + 1] - t[i + 1]
            if den != 0 and (i + 1) in N:
                lin = [Fraction(t[i + k + 1] - e, den), Fraction(-1, den)]
                acc = _padd(acc, _pmul(lin, N[i + 1]))
            newN[i] = acc
        N = newN
    return [N[a] for a in range(s - p, s + 1)]  # index a-e ↔ function e..e+p


@lru_cache(maxsize=None)
def exact_tables(p: int, n: int):
    """Exact M̂_ab = ∫N_aN_b and K̂_ab = ∫N'_aN'_b on integer knots, as dicts {(a,b): Fraction}."""
    m = n + p
    M = {}
    K = {}
    for e in range(n):
        B = element_basis(p, n, e)
        dB = [_pder(b) for b in B]
        for ia in range(p + 1):
            for ib in range(p + 1):
                a, b = e + ia, e + ib
                M[(a, b)] = M.get((a, b), Fraction(0)) + _pint01(_pmul(B[ia], B[ib]))
                K[(a, b)] = K.get((a, b), Fraction(0)) + _pint01(_pmul(dB[ia], dB[ib]))
    assert all(0 <= a < m and 0 <= b < m for a, b in M)
    return M, K


def banded_tables(p: int, n: int):
    """fp64 physical tables in band storage, shape (m, 2p+1): band[a, b-a+p].

    M1 = fl(fl(M̂)/n), K1 = fl(fl(K̂)·n)  (c.3; the rounding of each exact value is correct).
    Entries outside 0..m-1 are 0.
    """
    M, K = exact_tables(p, n)
    m = n + p
    Mb = np.zeros((m, 2 * p + 1))
    Kb = np.zeros((m, 2 * p + 1))
    for (a, b), v in M.items():
        Mb[a, b - a + p] = float(v) / float(n)
    for (a, b), v in K.items():
        Kb[a, b - a + p] = float(v) * float(n)
    return Mb, Kb


def hat_tables(p: int, n: int):
    """The rounded h=1 tables fl(M̂), fl(K̂) in band storage (for bitwise comparison with the library)."""
    M, K = exact_tables(p, n)
    m = n + p
    Mb = np.zeros((m, 2 * p + 1))
    Kb = np.zeros((m, 2 * p + 1))
    for (a, b), v in M.items():
        Mb[a, b - a + p] = float(v)
    for (a, b), v in K.items():
        Kb[a, b - a + p] = float(v)
    return Mb, Kb
