"""Per-level time of the V-cycle (exclusive ms per V-cycle, amg_get_level_times) for a workload at
1 or N GPUs (torchrun).  Runs without CUDA graphs (events between levels).

    AMG_GRAPHS=0 AMG_PROF_LEVELS=1 python tools/level_breakdown.py --config C3
    AMG_GRAPHS=0 AMG_PROF_LEVELS=1 torchrun --nproc-per-node 4 tools/level_breakdown.py --gpus 4
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import amg_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--per-rank-setup", action="store_true",
                    help="every rank builds the global hierarchy itself (no shared setup)")
    args = ap.parse_args()
    os.environ.setdefault("AMG_GRAPHS", "0")
    os.environ.setdefault("AMG_PROF_LEVELS", "1")
    import torch
    import torch.distributed as dist
    import paper_2511_21268_b200 as amg
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
    c = amg_inputs.CONFIGS[args.config]
    amg.set_num_threads(len(os.sched_getaffinity(0)))
    K, F = amg.iga_poisson(c["dim"], c["p"], c["n"], rhs=2, geometry=c.get("geometry", 0))
    prm = amg.params(c["p"], krylov=1, coarse_solver=1)
    if world > 1 and args.per_rank_setup:
        H = amg.Hierarchy(K, prm, dist=amg.make_dist(rank, world, device=int(os.environ.get("LOCAL_RANK", "0"))))
    elif world > 1:  # one host setup (rank 0), shares to every rank
        H = amg.setup_distributed(K if rank == 0 else None, prm, rank, world,
                                  device=int(os.environ.get("LOCAL_RANK", "0")))
    else:
        H = amg.Hierarchy(K, prm)
    b, e = H.local_rows()
    Fd = torch.from_numpy(np.ascontiguousarray(F[b:e])).cuda()
    H.solve(Fd)
    H.level_times()  # reset after the warm solve
    its = 0
    for _ in range(args.solves):
        its += H.solve(Fd)[1]
    t = H.level_times()
    out = {"rank": rank, "world": world, "transport": os.environ.get("AMG_TRANSPORT", "p2p"),
           "iters_per_solve": its / args.solves, "ms_per_vcycle_by_level": [round(v, 4) for v in t],
           "total_ms_per_vcycle": round(sum(t), 4), "levels_N": H.info()["N"],
           "ops": [[(lambda c: f'{c["layout"]}/{c["kernel"]}/G{c["G"]}U{c["U"]}')(H.op_config(l, k))
                    for k in range(3) if l + 1 < len(t) or k == 0] for l in range(len(t) - 1)]}
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, out)
        if rank == 0:
            for p_ in parts:
                print(json.dumps(p_), flush=True)
        dist.destroy_process_group()
    else:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
