"""Time the level operators (y = A x through amg_level_apply), one V-cycle and one solve for kernel
variants selected by environment (AMG_CSR_G, AMG_CSR_U) and amg_params.format.

    python tools/kernel_sweep.py --config C3 --variants "1:4:-,1:6:-,1:8:-,2:-:-"
variant = format:U:G ('-' = library default).  Prints one JSON line per variant.
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
    ap.add_argument("--variants", default="1:-:-")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2511_21268_b200 as amg
    c = amg_inputs.CONFIGS[args.config]
    K, F = amg.iga_poisson(c["dim"], c["p"], c["n"])
    Fd = torch.from_numpy(F).cuda()
    for var in args.variants.split(","):
        fmt, U, G = var.split(":")
        for key, val in (("AMG_CSR_U", U), ("AMG_CSR_G", G)):
            if val == "-":
                os.environ.pop(key, None)
            else:
                os.environ[key] = val
        t0 = time.perf_counter()
        H = amg.Hierarchy(K, amg.params(c["p"], format=int(fmt)))
        t_setup = time.perf_counter() - t0
        info = H.info()
        res = dict(variant=var, setup_s=round(t_setup, 1), levels=[])
        for l in range(info["levels"]):
            N = info["N"][l]
            x = torch.rand(N, dtype=torch.float64, device="cuda")
            y = torch.empty_like(x)
            for _ in range(3):
                H.apply(l, 0, x, y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                H.apply(l, 0, x, y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            byts = 12.0 * info["nnz"][l] + 24.0 * N
            res["levels"].append(dict(l=l, N=N, us=round(ms * 1e3, 1), GBps=round(byts / ms / 1e6, 1)))
        r = torch.rand(info["N"][0], dtype=torch.float64, device="cuda")
        for _ in range(2):
            H.vcycle(r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            H.vcycle(r)
        e1.record()
        torch.cuda.synchronize()
        res["vcycle_ms"] = round(e0.elapsed_time(e1) / 5, 3)
        u = torch.zeros_like(Fd)
        H.solve(Fd, u=u)
        u.zero_()
        torch.cuda.synchronize()
        e0.record()
        _, it, rr, _, st = H.solve(Fd, u=u)
        e1.record()
        torch.cuda.synchronize()
        res.update(solve_ms=round(e0.elapsed_time(e1), 2), iters=it)
        print(json.dumps(res), flush=True)
        H.close()
        del H
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
