"""Debug: distributed vs single-GPU V-cycle and PCG on a small cube (2 ranks, torchrun)."""
import os
import sys

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
dim, p, n = 3, 3, 12
K, F = amg.iga_poisson(dim, p, n)
for ml in (2, 3):
    prm = amg.params(p, max_levels=ml)
    H = amg.Hierarchy(K, prm, dist=amg.make_dist(rank, world, device=rank))
    b, e = H.local_rows()
    r = amg_inputs.uniform_pm1(K.shape[0], seed=3)
    z = H.vcycle(torch.from_numpy(np.ascontiguousarray(r[b:e])).cuda()).cpu().numpy()
    parts = [None] * world
    dist.all_gather_object(parts, (b, e, z))
    if rank == 0:
        zz = np.zeros(K.shape[0])
        for bb, ee, zl in parts:
            zz[bb:ee] = zl
        prm1 = amg.params(p, max_levels=ml)
        H1 = amg.Hierarchy(K, prm1)
        z1 = H1.vcycle(torch.from_numpy(r).cuda()).cpu().numpy()
        d = np.abs(zz - z1)
        print(f"max_levels={ml} levels={H1.info()['levels']} N={H1.info()['N']} vcycle max|diff|={d.max():.3e} "
              f"rel={d.max() / np.abs(z1).max():.3e} worst rows {np.argsort(-d)[:8].tolist()} split={parts[0][1]}",
              flush=True)
    dist.barrier()
    del H
dist.destroy_process_group()
