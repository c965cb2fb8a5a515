"""Debug: distributed vs single-GPU PCG iteration counts on a small cube (2 ranks, torchrun)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2511_21268_b200 as amg  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
for solver in ("pcg", "fcg"):
    K, F = amg.iga_poisson(3, 3, 12, rhs=2 if solver == "fcg" else 0)
    kw = dict(krylov=1, coarse_solver=1) if solver == "fcg" else {}
    H = amg.Hierarchy(K, amg.params(3, **kw), dist=amg.make_dist(rank, world, device=rank))
    b, e = H.local_rows()
    Fl = torch.from_numpy(np.ascontiguousarray(F[b:e])).cuda()
    if os.environ.get("DBG_VCYCLE_FIRST") == "1":
        zv = H.vcycle(Fl.clone())
        torch.cuda.synchronize()
    if os.environ.get("DBG_GATHER") == "1":
        zz = H.vcycle(Fl.clone()).cpu().numpy()
        parts = [None] * world
        dist.all_gather_object(parts, (b, e, zz))
    u0 = torch.zeros_like(Fl)
    print(f"rank {rank}: |F|={Fl.norm().item():.6e} |u0|={u0.norm().item():.3e} dev={torch.cuda.current_device()}", flush=True)
    u, it, rr, hist, st = H.solve(Fl, rtol=1e-6)
    if rank == 0:
        H1 = amg.Hierarchy(K, amg.params(3, **kw))
        u1, it1, rr1, hist1, st1 = H1.solve(torch.from_numpy(F).cuda(), rtol=1e-6)
        print(f"{solver}: dist iters={it} st={st} hist[:4]={np.round(hist[:4], 6).tolist()} | single iters={it1} "
              f"hist[:4]={np.round(hist1[:4], 6).tolist()}", flush=True)
    dist.barrier()
    del H
dist.destroy_process_group()
