"""Multi-GPU host logic on the CPU: world_size-2 gloo processes build the same hierarchy, take their
row blocks and halo plans from the library (amg_dist_view_get), exchange ghost values over gloo exactly
as the device path does over NCCL, and check

* the row blocks of every level tile [0, N_l) contiguously;
* every local row maps back (owned / ghost column numbering) to the global row, bitwise;
* the halo exchange delivers exactly x[ghost ids];
* the distributed product equals the global product on every owned row.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, rep_nnz, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        os.environ["AMG_REPLICATE_NNZ"] = str(rep_nnz)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2511_21268_b200 as amg
        import amg_inputs
        dim, p, n = case[:3]
        geom = case[3] if len(case) > 3 else 0  # 2: the three-patch L-shape
        K, F = amg.iga_poisson(dim, p, n, rhs=1 if geom else 0, geometry=geom)
        H = amg.Hierarchy(K, amg.params(p, host_only=1), dist=amg.make_dist(rank, world, nccl_id=bytes(128)))
        info = H.info()
        checked = 0
        for l in range(info["levels"]):
            e = H.export(l)
            Kg = e["K"].to_scipy()
            ops = [(0, Kg)]
            if e["P"] is not None:
                Pg = e["P"].to_scipy()
                ops += [(1, Pg), (2, Pg.T.tocsr())]
            for op, A in ops:
                v = H.dist_view(l, op)
                if v["replicated"]:
                    continue
                # row blocks tile the level
                rb = torch.tensor([v["row_begin"], v["row_end"]], dtype=torch.int64)
                allb = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(allb, rb)
                allb = [t.tolist() for t in allb]
                assert allb[0][0] == 0 and allb[-1][1] == A.shape[0]
                assert all(allb[k][1] == allb[k + 1][0] for k in range(world - 1))
                loc = v["local"]
                nown = v["col_end"] - v["col_begin"]
                ghost = v["ghost"]
                # local -> global column map reproduces the global rows bitwise
                nlo = v["n_ghost_lo"]
                if v["full_cols"]:
                    gmap, shift = np.arange(A.shape[1]), 0
                else:  # local index li -> gmap[li + nlo]: [lower ghosts | owned | upper ghosts]
                    gmap = np.concatenate([ghost[:nlo], np.arange(v["col_begin"], v["col_end"]), ghost[nlo:]])
                    shift = nlo
                    assert np.all(ghost[:nlo] < v["col_begin"]) and np.all(ghost[nlo:] >= v["col_end"])
                Ar = A[v["row_begin"]:v["row_end"]]
                assert np.array_equal(gmap[loc.indices + shift], Ar.indices) and np.array_equal(loc.indptr, Ar.indptr)
                # global order kept: every local row is ascending
                assert all(np.all(np.diff(loc.indices[loc.indptr[i]:loc.indptr[i + 1]]) > 0) for i in range(loc.shape[0]))
                assert np.array_equal(loc.data.view(np.uint64), Ar.data.view(np.uint64))
                # halo exchange over gloo
                x = amg_inputs.uniform_pm1(A.shape[1], seed=100 + 10 * l + op)
                if v["full_cols"]:
                    xl = x
                else:
                    xown = x[v["col_begin"]:v["col_end"]]
                    ghosts = np.full(len(ghost), np.nan)
                    reqs, bufs = [], []
                    for r in range(world):
                        if r == rank:
                            continue
                        s0, sc = v["send_off"][r], v["send_count"][r]
                        sb = torch.from_numpy(np.ascontiguousarray(xown[v["send_idx"][s0:s0 + sc]]))
                        rbuf = torch.zeros(int(v["recv_count"][r]), dtype=torch.float64)
                        if sc:
                            reqs.append(dist.isend(sb, r))
                        if len(rbuf):
                            reqs.append(dist.irecv(rbuf, r))
                        bufs.append((r, rbuf, sb))
                    for rq in reqs:
                        rq.wait()
                    for r, rbuf, _ in bufs:
                        o = v["recv_off"][r]
                        ghosts[o:o + len(rbuf)] = rbuf.numpy()
                    assert np.array_equal(ghosts, x[ghost])
                    xl = np.concatenate([ghosts[:nlo], xown, ghosts[nlo:]])
                y = np.array([np.dot(loc.data[loc.indptr[i]:loc.indptr[i + 1]],
                                     xl[loc.indices[loc.indptr[i]:loc.indptr[i + 1]] + shift])
                              for i in range(loc.shape[0])]) if loc.shape[0] else np.zeros(0)
                yref = Ar @ x
                assert np.abs(y - yref).max() <= 1e-14 * (abs(Ar) @ np.abs(x)).max()
                checked += 1
        dist.barrier()
        q.put((rank, "ok", checked))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("case,rep_nnz", [((3, 2, 12), 1000), ((3, 3, 10), 20000), ((2, 2, 16), 100),
                                           ((3, 2, 6, 2), 1000)])
def test_partition_and_halo_plans_world2(case, rep_nnz):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, rep_nnz, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, status, detail in res:
        assert status == "ok", detail
        assert detail >= 3  # at least K_0, P̄_0, R_0 were distributed and checked


# ---- shared setup: one host hierarchy, one share per rank (amg_share_export / amg_setup_from_share) ----

def _views(H, levels):
    out = {}
    for l in range(levels):
        for op in range(3 if l + 1 < levels else 1):
            v = H.dist_view(l, op)
            if v["replicated"]:
                out[(l, op)] = "replicated"
                continue
            loc = v.pop("local")
            v = {k: (np.asarray(x).copy() if isinstance(x, np.ndarray) else x) for k, x in v.items()}
            v["local"] = (loc.indptr.copy(), loc.indices.copy(), loc.data.view(np.uint64).copy())
            out[(l, op)] = v
    return out


def _same(a, b):
    assert a.keys() == b.keys()
    for key in a:
        va, vb = a[key], b[key]
        if isinstance(va, str) or isinstance(vb, str):
            assert va == vb, key
            continue
        assert va.keys() == vb.keys(), key
        for f in va:
            if f == "local":
                assert all(np.array_equal(x, y) for x, y in zip(va[f], vb[f])), (key, f)
            else:
                assert np.array_equal(np.asarray(va[f]), np.asarray(vb[f])), (key, f)


@pytest.mark.parametrize("case,world,rep_nnz", [((3, 2, 12), 2, 1000), ((3, 3, 10), 3, 20000),
                                                ((2, 2, 16), 4, 100), ((3, 2, 6, 2), 2, 1000)])
def test_share_equals_per_rank_setup(case, world, rep_nnz, monkeypatch):
    """A rank's hierarchy rebuilt from its share has exactly the plan, local operators (bitwise values)
    and sizes that amg_setup with that rank's amg_dist builds from the full K."""
    monkeypatch.setenv("AMG_REPLICATE_NNZ", str(rep_nnz))
    import paper_2511_21268_b200 as amg
    dim, p, n = case[:3]
    geom = case[3] if len(case) > 3 else 0
    K, _ = amg.iga_poisson(dim, p, n, rhs=1 if geom else 0, geometry=geom)
    G = amg.Hierarchy(K, amg.params(p, host_only=1))
    for r in range(world):
        d = amg.make_dist(r, world, nccl_id=bytes(128))
        ref = amg.Hierarchy(K, amg.params(p, host_only=1), dist=d)
        sh = G.export_share(r, world)
        H = amg.Hierarchy.from_share(sh, d, host_only=True)
        sh.close()
        assert H.info() == ref.info() == G.info()
        assert H.local_rows() == ref.local_rows()
        L = ref.info()["levels"]
        _same(_views(H, L), _views(ref, L))
        with pytest.raises(amg.AmgError):
            H.export(0)  # the global operators are not held
        with pytest.raises(amg.AmgError):
            H.export_share(0, world)


def test_share_rejects_wrong_rank_and_corruption():
    import paper_2511_21268_b200 as amg
    K, _ = amg.iga_poisson(2, 2, 8)
    G = amg.Hierarchy(K, amg.params(2, host_only=1))
    sh = G.export_share(1, 2)
    blob = sh.array.copy()
    sh.close()
    with pytest.raises(amg.AmgError):
        amg.Hierarchy.from_share(blob, amg.make_dist(0, 2, nccl_id=bytes(128)), host_only=True)
    with pytest.raises(amg.AmgError):
        amg.Hierarchy.from_share(blob[:-9], amg.make_dist(1, 2, nccl_id=bytes(128)), host_only=True)
    bad = blob.copy()
    bad[0] ^= 1
    with pytest.raises(amg.AmgError):
        amg.Hierarchy.from_share(bad, amg.make_dist(1, 2, nccl_id=bytes(128)), host_only=True)
    with pytest.raises(amg.AmgError):
        G.export_share(2, 2)
    # one rank: the whole hierarchy, every level "replicated"
    sh1 = G.export_share(0, 1)
    H1 = amg.Hierarchy.from_share(sh1, None, host_only=True)
    assert H1.info() == G.info()


def _share_worker(rank, world, port, case, rep_nnz, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        os.environ["AMG_REPLICATE_NNZ"] = str(rep_nnz)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2511_21268_b200 as amg
        dim, p, n = case
        K, _ = amg.iga_poisson(dim, p, n)
        prm = amg.params(p, host_only=1)
        # small chunks: the blob crosses several sends
        H = amg.setup_distributed(K if rank == 0 else None, prm, rank, world, nccl_id=bytes(128),
                                  host_only=True, group=dist.group.WORLD, chunk_bytes=4096)
        ref = amg.Hierarchy(K, prm, dist=amg.make_dist(rank, world, nccl_id=bytes(128)))
        assert H.info() == ref.info()
        L = ref.info()["levels"]
        _same(_views(H, L), _views(ref, L))
        dist.barrier()
        q.put((rank, "ok", L))
    except Exception:  # noqa: BLE001
        import traceback
        q.put((rank, "fail", traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_setup_distributed_world2():
    """setup_distributed over gloo: rank 0 builds once and ships rank 1 its share in chunks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_share_worker, args=(r, 2, port, (3, 2, 12), 1000, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, status, detail in res:
        assert status == "ok", detail
