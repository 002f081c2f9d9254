"""The NCCL transport of the row-partitioned path on >= 2 GPUs (one process per GPU, torch.distributed NCCL for
the id broadcast, wl_comm_create): skipped on a single-GPU box, where tests/test_gpu_multirank.py runs the same
code path through the loopback transport.  Each rank builds its row block (wl_partition), applies 𝕃 for
θ ∈ {1, 0.5, 0} (halo exchange with the A_loc/A_halo overlap, allreduced Gram sums) and diffuses; rank 0 gathers
the blocks and compares them with the single-GPU operator and the series oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import graphgen as gg
    import paper_2601_11338_b200 as wl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        g = gg.rmat(13, 6000, 60000, seed=21, perm_seed=22)
        bounds = wl.partition(g.row_ptr, world)
        rb, re = int(bounds[rank]), int(bounds[rank + 1])
        rp = g.row_ptr[rb:re + 1]
        ci = g.col_idx[rp[0]:rp[-1]]
        comm = wl.Comm(rank, world, rank)
        beta = 0.05
        V = gg.vectors(g.n, 2, 77)
        op = wl.Operator(g.n, rp, ci, row_range=(rb, re), comm=comm, thetas=[1.0, 0.5, 0.0], f=("exp", beta))
        LV = op.apply(torch.from_numpy(V[rb:re].copy()).cuda()).cpu().numpy()
        X = op.diffuse(torch.from_numpy(np.ascontiguousarray(V[rb:re, 0])).cuda(), [0.5, 2.0], k_out=30).cpu().numpy()
        op.close()
        comm.close()
        parts = [None] * world
        dist.all_gather_object(parts, (LV, X))
        if rank == 0:
            op1 = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0, 0.5, 0.0], f=("exp", beta))
            L1 = op1.apply(torch.from_numpy(V).cuda()).cpu().numpy()
            X1 = op1.diffuse(torch.from_numpy(np.ascontiguousarray(V[:, 0])).cuda(), [0.5, 2.0], k_out=30).cpu().numpy()
            op1.close()
            LVa = np.vstack([p[0] for p in parts])
            Xa = np.vstack([p[1] for p in parts])
            q.put((float(np.max(np.linalg.norm(LVa - L1, axis=0) / np.linalg.norm(L1, axis=0))),
                   float(np.max(np.linalg.norm(Xa - X1, axis=0) / np.linalg.norm(X1, axis=0)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_nccl_two_gpus_vs_one():
    import torch.multiprocessing as mp
    from paper_2601_11338_b200 import build
    build.build()
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs)
    e_apply, e_diff = q.get(timeout=10)
    assert e_apply < 1e-12 and e_diff < 1e-12
