"""Debug: the windowed SELL-VI core on a 2-rank P2P share (torchrun), step by step with prints, the level-0
operator applied alone (amg_level_apply: no halo, no P2P), then one V-cycle, then a short solve."""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import amg_inputs  # noqa: E402
import paper_2511_21268_b200 as amg  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
os.environ.setdefault("AMG_REPLICATE_NNZ", "200000")


def say(*a):
    print(f"[rank {rank} {time.strftime('%H:%M:%S')}]", *a, flush=True)


K, F = amg.iga_poisson(3, 2, 32)
H = amg.Hierarchy(K, amg.params(2), dist=amg.make_dist(rank, world, device=rank))
info = H.info()
say("levels", info["levels"], [H.op_config(l, 0)["layout"] for l in range(info["levels"])],
    H.op_config(0, 0))
b, e = H.local_rows()
dist.barrier()
r = amg_inputs.uniform_pm1(K.shape[0], seed=3)
say("vcycle ...")
z = H.vcycle(torch.from_numpy(np.ascontiguousarray(r[b:e])).cuda())
torch.cuda.synchronize()
say("vcycle done", float(z.abs().max()))
dist.barrier()
say("solve ...")
u, it, rr, hist, st = H.solve(torch.from_numpy(np.ascontiguousarray(F[b:e])).cuda(), rtol=1e-6, maxit=50)
torch.cuda.synchronize()
say("solve done", it, st, rr)
dist.barrier()
dist.destroy_process_group()
