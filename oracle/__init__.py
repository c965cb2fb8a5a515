"""Oracle: a plain, slow, obviously-correct CPU implementation of the paper's method.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import, call, link or execute anything under
``oracle/``.  The product (``paper_2511_21268_b200``) never imports it and shares no code with it:
no kernels, headers, helpers, tables or constant generators.  The only module both sides use is
``amg_inputs`` (seeded random numbers and workload names, no arithmetic of the method).

Contents (each function cites the PAPER.md passage it follows):
  * ``tables.py``  — exact rational 1-D mass/stiffness tables (c.3);
  * ``bspline.py`` — float Cox–de Boor, Gauss quadrature, a genuine d-D element-loop assembly
    (independent cross-check of c.4), the manufactured load vector (c.5) and L2 error;
  * ``oracle.c``   — Kronecker assembly (c.4), compatible weighted matching + aggregation +
    smoothed prolongator + Galerkin RAP (c.6-c.15), Chebyshev-ℓ1-Jacobi V-cycle (c.16-c.18) and
    PCG (c.19), single-threaded, ``-O2 -ffp-contract=off``;
  * ``core.py``    — ctypes wrapper returning numpy / scipy objects;
  * ``cube_paper.py`` — the paper's cube data (NEXT-1): projected Dirichlet data, Neumann loads, lifting;
  * ``ring.py``    — the thick quarter ring (NEXT-3): NURBS map, weighted tables, its data;
  * ``lshape.py``  — the three-patch L-shape (NEXT-4): conforming gluing, its data.

Parity status of each function (pins in tests/test_oracle_*.py) is listed in DESIGN.md §4.
"""
from .core import (  # noqa: F401
    OParams,
    OHierarchy,
    assemble,
    build_liboracle,
    cij,
    fcg,
    galerkin_pairwise,
    pairwise,
    pcg,
    setup,
    smooth,
    spmv,
    vcycle,
)
