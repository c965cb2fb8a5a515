"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no B-splines, no matching, no smoothing).
It only names the workloads of BASELINE.json ``configs`` and draws seeded random numbers,
so that the oracle (``oracle/``) and the CUDA library (``paper_2511_21268_b200``) can be fed
identical inputs without sharing any code with each other.

Workloads (PAPER.md P:L1061-1072 for the cube boundary convention:
Dirichlet on sides 1,2,3 = {x=0, x=1, y=0}, Neumann on sides 4,5,6):

=====  ===  ===  ====  =====================================================
name   dim  p    n     role
=====  ===  ===  ====  =====================================================
C1     2    2    16    oracle-sized case (seconds)
C2     3    2    32    single-B200 full hierarchy, parity at full size
C3     3    3    96    the paper's GPU cube case (Table 1b k=96: 941,094 DOFs)
C4     3    4    128   high-degree bandwidth stress
C5     3    2    250+  weak scaling, ~16M DOFs per GPU (n = 250/315/398/502)
C5s    3    2    158+  weak scaling, ~4M DOFs per GPU (n = 158/200/252/317)
R3     3    3    96    thick quarter ring (NEXT-3, Table 3)
R4     3    4    96    thick quarter ring, the paper's GPU ring case
L3     3    3    96    three-patch L-shape, the paper's GPU multipatch case (NEXT-4, Table 2)
=====  ===  ===  ====  =====================================================
"""
from __future__ import annotations

import numpy as np

# bit s-1 set <=> side s is Dirichlet; sides 1:x=0 2:x=1 3:y=0 4:y=1 5:z=0 6:z=1
DIRICHLET_123 = 0b000111

CONFIGS = {
    "C1": dict(dim=2, p=2, n=16),
    "C2": dict(dim=3, p=2, n=32),
    "C3": dict(dim=3, p=3, n=96),
    "C4": dict(dim=3, p=4, n=128),
    "C5": dict(dim=3, p=2, n=250),
    # C5 at a quarter of the per-GPU size (≈ 4M DOFs per GPU): the weak-scaling series that fits one
    # global host setup in the GPU box's host RAM at 2 and 4 GPUs
    "C5s": dict(dim=3, p=2, n=158),
    # NEXT-3: the thick quarter ring, Table 3 k=96 p=3 (941,094 DOFs); seeded random RHS
    "R3": dict(dim=3, p=3, n=96, geometry=1),
    # the paper's GPU ring case (k=96 p=4, 970,200 DOFs; 6.234 s on one A30)
    "R4": dict(dim=3, p=4, n=96, geometry=1),
    # NEXT-4: the three-patch L-shape, the paper's GPU multipatch case (P:L2674,
    # L2779: k=96 p=3, Table 2b 2,775,752 DOFs; 4.636 s on one A30); the paper's L-shape data
    "L3": dict(dim=3, p=3, n=96, geometry=2),
}
C5_WEAK_N = {1: 250, 2: 315, 4: 398, 8: 502}
C5S_WEAK_N = {1: 158, 2: 200, 4: 252, 8: 317}

# Chebyshev degree by spline degree: P:L1117 (deg_3=8, deg_4=12, deg_5=14, deg_6=16);
# p=2 is unstated in the paper -> 4 (SURVEY c.16); p=1 -> 2.
CHEB_DEGREE = {1: 2, 2: 4, 3: 8, 4: 12, 5: 14, 6: 16}

SEED = 20251121


def free_dofs(dim: int, p: int, n: int, dirichlet_sides: int = DIRICHLET_123) -> int:
    """Count of free DOFs: (n+p) functions per axis minus the Dirichlet-side layers.

    Pure counting (no method arithmetic); used to size buffers before calling either side.
    """
    m = n + p
    total = 1
    for ax in range(dim):
        lo = 1 if dirichlet_sides >> (2 * ax) & 1 else 0
        hi = 1 if dirichlet_sides >> (2 * ax + 1) & 1 else 0
        total *= m - lo - hi
    return total


_MASK64 = (1 << 64) - 1


def splitmix64(seed: int, count: int) -> np.ndarray:
    """Counter-based splitmix64 stream (Steele, Lea, Flood 2014) as uint64, vectorised."""
    idx = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & _MASK64) + idx * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(count: int, seed: int = SEED) -> np.ndarray:
    """Seeded uniform(-1, 1) fp64 vector (53 random bits per value)."""
    u = (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    return 2.0 * u - 1.0
