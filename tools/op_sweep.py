"""Time y = A·x (amg_level_apply) for every CSR kernel configuration of the large operators.

    python tools/op_sweep.py --config C3 [--levels 0,1,2] [--reps 10]
One JSON line per (level, op, kernel, G, U): µs per application and GB/s of the format's own streamed
bytes (alg_bytes of amg_operator_config + 16 B/row for the x gather and the y write).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import amg_inputs  # noqa: E402


def kind_name(k: int) -> str:
    return ("csr_tma" if k & 1 else "csr_regs") + ("_d16" if k & 2 else "") + ("_vi" if k & 8 else "") + \
        ("_pf" if k & 4 else "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--levels", default="0,1,2")
    ap.add_argument("--ops", default="0")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--sell", action="store_true", help="also time the SELL-32 layout")
    ap.add_argument("--format", type=int, default=0, help="amg_params.format of the swept hierarchy")
    ap.add_argument("--n", type=int, default=0, help="override the config's elements per direction")
    args = ap.parse_args()
    import torch
    import paper_2511_21268_b200 as amg
    c = dict(amg_inputs.CONFIGS[args.config])
    if args.n:
        c["n"] = args.n
    K, F = amg.iga_poisson(c["dim"], c["p"], c["n"])
    H = amg.Hierarchy(K, amg.params(c["p"], format=args.format))
    del K
    info = H.info()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for l in map(int, args.levels.split(",")):
        for op in map(int, args.ops.split(",")):
            if op > 0 and l + 1 >= info["levels"]:
                continue
            chosen = H.op_config(l, op)
            nr = info["N"][l] if op < 2 else info["N"][l + 1]
            ncol = info["N"][l] if op != 1 else info["N"][l + 1]
            x = torch.rand(ncol, dtype=torch.float64, device="cuda")
            y = torch.empty(nr, dtype=torch.float64, device="cuda")
            kerns = [0, 1, 2, 3, 4, 6]  # bit 0 TMA, bit 1 16-bit columns, bit 2 L2 prefetch, bit 3 value index
            if chosen["n_values"]:
                kerns += [8, 10, 12, 14]
            sellvi = chosen["layout"] in ("sellvi", "sellviw")
            sk = [1, 2] if chosen["layout"] == "sellviw" else [0]  # windowed: windows staged per CTA
            for kern in (sk if sellvi else kerns):
                for G in ((32,) if sellvi else (1, 2, 4, 8, 32)):
                    for U in ((1, 2, 4) if sellvi else (2, 4, 6, 8)):
                        if (kern & 1) and U > 4:
                            continue
                        try:
                            H.set_op_config(l, op, kern, G, U)
                        except Exception:  # noqa: BLE001
                            continue
                        H.apply(l, op, x, y)
                        torch.cuda.synchronize()
                        e0.record()
                        for _ in range(args.reps):
                            H.apply(l, op, x, y)
                        e1.record()
                        torch.cuda.synchronize()
                        us = e0.elapsed_time(e1) * 1e3 / args.reps
                        cfg = H.op_config(l, op)
                        gbs = (cfg["alg_bytes"] + 16.0 * nr) / (us * 1e-6) / 1e9
                        print(json.dumps(dict(level=l, op=op, kernel=(chosen["layout"] + (f"_b{kern}" if kern else "")) if sellvi else kind_name(kern), G=G, U=U, us=round(us, 1),
                                              GBps=round(gbs, 1), alg_bytes=cfg["alg_bytes"])), flush=True)
            H.set_op_config(l, op, chosen["kernel_bits"], chosen["G"], chosen["U"])
            print(json.dumps(dict(level=l, op=op, autotuned=chosen)), flush=True)
    if args.sell:  # the SELL-32 layout (one row per lane) of the same operators
        H = None
        K, F = amg.iga_poisson(c["dim"], c["p"], c["n"])
        H = amg.Hierarchy(K, amg.params(c["p"], format=2))
        del K
        for l in map(int, args.levels.split(",")):
            for op in map(int, args.ops.split(",")):
                if op > 0 and l + 1 >= info["levels"]:
                    continue
                nr = info["N"][l] if op < 2 else info["N"][l + 1]
                ncol = info["N"][l] if op != 1 else info["N"][l + 1]
                x = torch.rand(ncol, dtype=torch.float64, device="cuda")
                y = torch.empty(nr, dtype=torch.float64, device="cuda")
                H.apply(l, op, x, y)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(args.reps):
                    H.apply(l, op, x, y)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / args.reps
                cfg = H.op_config(l, op)
                gbs = (cfg["alg_bytes"] + 16.0 * nr) / (us * 1e-6) / 1e9
                print(json.dumps(dict(level=l, op=op, kernel="sell32", us=round(us, 1), GBps=round(gbs, 1),
                                      stored=cfg["stored"], nnz=cfg["nnz"])), flush=True)


if __name__ == "__main__":
    main()
