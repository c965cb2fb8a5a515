"""Write the oracle's hierarchy sizes (N, nnz, nnz(P̄) per level), setup time, PCG iteration count
and solve time for a workload (manufactured RHS, rtol 1e-6), and the FCG iteration count / solve time
of the paper's own cube experiment (its data, FCG, §5.1 coarse CG).

TEST INFRASTRUCTURE (oracle only): calls nothing but oracle/.  Output: oracle/sizes_<cfg>.json, read
by bench.py's reference arm for the byte model (a full oracle setup of C3 takes minutes).

    python oracle/scripts/hierarchy_sizes.py C3
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import amg_inputs  # noqa: E402
import oracle  # noqa: E402


def main(cfg: str) -> None:
    c = amg_inputs.CONFIGS[cfg]
    t0 = time.perf_counter()
    K = oracle.assemble(c["dim"], c["p"], c["n"])
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    H = oracle.setup(K, oracle.OParams.for_degree(c["p"]))
    t_setup = time.perf_counter() - t0
    from oracle import bspline
    F = bspline.load_vector(c["dim"], c["p"], c["n"])
    t0 = time.perf_counter()
    u, iters, relres, hist, rc = oracle.pcg(H, F, rtol=1e-6, maxit=200)
    t_solve = time.perf_counter() - t0
    # the paper's own experiment: its data, FCG, §5.1 coarse CG
    paper = {}
    if c["dim"] == 3:
        from oracle import cube_paper
        Fp, _ = cube_paper.paper_cube_rhs(c["p"], c["n"])
        H2 = oracle.setup(K, oracle.OParams.for_degree(c["p"], coarse_solver=1))
        t0 = time.perf_counter()
        u2, it2, rr2, h2, rc2 = oracle.fcg(H2, Fp, rtol=1e-6, maxit=200)
        # the converged iterate (the it2-th) sampled every 997th row (+ the last row) and the residual
        # history, for the full-size GPU parity test (tests/test_gpu_parity.py::test_c3_paper_solve_vs_oracle_artifact)
        idx = list(range(0, len(u2), 997)) + [len(u2) - 1]
        paper = dict(oracle_iters_paper=it2, oracle_relres_paper=rr2,
                     oracle_solve_paper_s=round(time.perf_counter() - t0, 2),
                     oracle_hist_paper=[float(h) for h in h2], u_sample_stride=997,
                     u_sample_paper=[float(u2[i]) for i in idx], u_norm_paper=float(np.linalg.norm(u2)))
    out = dict(workload=cfg, oracle_iters=iters, oracle_relres=relres, oracle_solve_s=round(t_solve, 2), **paper,
               levels=H.nlevels, N=[L.N for L in H.levels], nnz=[L.K.nnz for L in H.levels],
               nnz_P=[(L.P.nnz if L.P is not None else 0) for L in H.levels], opc=H.opc(),
               oracle_assemble_s=round(t_asm, 2), oracle_setup_s=round(t_setup, 2), threads=1)
    with open(os.path.join(ROOT, "oracle", f"sizes_{cfg}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3")
