"""The oracle, as it stands, timed on this host: bench.py's `cpu_baseline` and `--impl reference` leg.

TEST INFRASTRUCTURE (oracle only): imports nothing but oracle/ and amg_inputs (seeded inputs).  The
workload's system is assembled, its right-hand side built and its hierarchy set up by the ORACLE
(single-threaded plain C + Python), then its FCG (the paper's experiment: its data, FCG P:L1107, §5.1
coarse CG P:L1114) or PCG (manufactured problem) runs and every iteration is timed on its own
(`or_fcg_cb` observer: clock reads only).  One STEP = one Krylov iteration (all §8(a) rows once:
SpMV + dots + updates + one V-cycle), the unit bench.py's GPU arm times; a solve that converges is
restarted from u0 = 0, so `--warmup W --steps K` runs exactly W + K iterations.

    python oracle/scripts/cpu_baseline.py --config C3 --warmup 0 --steps 2 [--problem paper] [--full-solve]
Prints one JSON line: setup/assembly times, per-step times, s_per_iter, the CPU model and cores used.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import resource
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import amg_inputs  # noqa: E402
import oracle  # noqa: E402


def cpu_model() -> dict:
    model, sockets, cores = platform.processor() or "unknown", None, None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = dict(l.split(":", 1) for l in out.splitlines() if ":" in l)
        kv = {k.strip(): v.strip() for k, v in kv.items()}
        model = kv.get("Model name", model)
        sockets = kv.get("Socket(s)")
        cores = kv.get("CPU(s)")
    except Exception:  # noqa: BLE001
        pass
    mem = None
    try:
        with open("/proc/meminfo") as f:
            mem = round(int(f.readline().split()[1]) / 2 ** 20, 1)
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "sockets": sockets, "host_cpus": cores, "host_mem_gib": mem}


def build_problem(cfg: str, problem: str):
    """K and F of the workload, by the oracle only."""
    c = amg_inputs.CONFIGS[cfg]
    dim, p, n, geom = c["dim"], c["p"], c["n"], c.get("geometry", 0)
    paper = problem == "paper" and dim == 3
    if geom == 1:
        from oracle import ring
        K = ring.assemble_ring(p, n)
        F = ring.paper_ring_rhs(p, n)[0] if paper else amg_inputs.uniform_pm1(K.shape[0], seed=amg_inputs.SEED)
    elif geom == 2:
        from oracle import lshape
        K = lshape.assemble_lshape(p, n)
        F = lshape.paper_lshape_rhs(p, n)[0] if paper else amg_inputs.uniform_pm1(K.shape[0], seed=amg_inputs.SEED)
    else:
        K = oracle.assemble(dim, p, n)
        if paper:
            from oracle import cube_paper
            F = cube_paper.paper_cube_rhs(p, n)[0]
        else:
            from oracle import bspline
            F = bspline.load_vector(dim, p, n)
    return K, np.ascontiguousarray(F, dtype=np.float64), paper


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--problem", default="paper", choices=["paper", "manufactured"])
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--full-solve", action="store_true", help="also run one full solve (iteration count)")
    args = ap.parse_args()
    c = amg_inputs.CONFIGS[args.config]
    t0 = time.perf_counter()
    K, F, paper = build_problem(args.config, args.problem)
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    H = oracle.setup(K, oracle.OParams.for_degree(c["p"], coarse_solver=1 if paper else 0))
    t_setup = time.perf_counter() - t0
    del K
    krylov = oracle.fcg if paper else oracle.pcg
    full = None
    if args.full_solve:
        t0 = time.perf_counter()
        u, it, rr, hist, rc = krylov(H, F, rtol=1e-6, maxit=200)
        full = dict(iters=it, relres=rr, rc=rc, solve_s=round(time.perf_counter() - t0, 3))
    total = args.warmup + args.steps
    times: list[float] = []
    while len(times) < total:
        need = total - len(times)
        stamps = [time.perf_counter()]
        if paper:
            def observer(k: int) -> bool:
                stamps.append(time.perf_counter())
                return len(stamps) - 1 >= need  # stop before the next iteration's V-cycle

            u, it, rr, hist, rc = oracle.fcg(H, F, rtol=1e-6, maxit=need, observer=observer)
            if len(stamps) - 1 < it:  # the converged iteration calls no observer
                stamps.append(time.perf_counter())
            times += [b - a for a, b in zip(stamps[:-1], stamps[1:])]
        else:  # or_pcg has no observer: whole solves of the remaining budget, per iteration
            u, it, rr, hist, rc = oracle.pcg(H, F, rtol=1e-6, maxit=need)
            times += [(time.perf_counter() - stamps[0]) / max(it, 1)] * max(it, 1)
    timed = times[args.warmup:]
    s_iter = sum(timed) / max(len(timed), 1)
    out = dict(config=args.config, problem="paper" if paper else "manufactured", krylov="FCG(1)" if paper else "PCG",
               N=H.levels[0].N, levels=H.nlevels, opc=round(H.opc(), 4),
               assemble_s=round(t_asm, 2), setup_s=round(t_setup, 2), step_s=[round(t, 4) for t in timed],
               warmup=args.warmup, steps=args.steps, s_per_iter=round(s_iter, 4), full_solve=full,
               threads=1, max_rss_gib=round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2 ** 20, 2),
               **cpu_model())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
