"""Profiling driver: set up a workload, run warm-up solves, then `--solves` solves (for ncu / sanitizer).

    python tools/profile_solve.py --config C3 --warm 1 --solves 1
Prints one JSON line with the library's own kernel-launch count per solve (to compute ncu -s / -c).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import amg_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--warm", type=int, default=1)
    ap.add_argument("--solves", type=int, default=1)
    ap.add_argument("--format", type=int, default=0)
    args = ap.parse_args()
    import torch
    import paper_2511_21268_b200 as amg
    os.environ.setdefault("AMG_TUNE_CACHE", os.path.join(ROOT, "profiles", f"tune_{args.config}.txt"))
    c = amg_inputs.CONFIGS[args.config]
    geom = c.get("geometry", 0)
    K, F = amg.iga_poisson(c["dim"], c["p"], c["n"], rhs=2 if geom else 0, geometry=geom)
    H = amg.Hierarchy(K, amg.params(c["p"], format=args.format))
    Fd = torch.from_numpy(F).cuda()
    u = torch.zeros_like(Fd)
    H.set_profiling(True)
    for _ in range(args.warm):
        u.zero_()
        H.solve(Fd, u=u)
    torch.cuda.synchronize()
    warm_launches = H.kernel_stats()["kernels_launched"]
    t0 = time.perf_counter()
    its = []
    torch.cuda.nvtx.range_push("solve")  # ncu --nvtx --nvtx-include "solve/" skips setup/autotuning
    for _ in range(args.solves):
        u.zero_()
        its.append(H.solve(Fd, u=u)[1])
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ks = H.kernel_stats()
    ops = [H.op_config(l, 0) for l in range(H.info()["levels"])]
    print(json.dumps(dict(config=args.config, info=H.info(), iters=its, warm_launches=warm_launches, level_ops=ops,
                          launches_per_solve=(ks["kernels_launched"] - warm_launches) // max(args.solves, 1),
                          wall_s_per_solve=dt / max(args.solves, 1))))


if __name__ == "__main__":
    main()
