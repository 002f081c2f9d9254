"""N>1 host logic on CPU (gloo, world_size 2 and 3): the nnz-balanced row partition and the halo
plan of the C library (wl_partition, wl_halo_plan), driven through the same request/response
exchange the NCCL path performs (owners pack the rows peers ask for), must reproduce the global
SpMV A x row block by row block, and the per-rank Gram partial sums must allreduce to the global
dot products (the allreduce of Krylov inner products)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen as gg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, qout):
    import torch
    import paper_2601_11338_b200 as wl
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = gg.rmat(12, 3000, 25000, seed=11, perm_seed=12)
        bounds = wl.partition(g.row_ptr, world)
        rb, re = int(bounds[rank]), int(bounds[rank + 1])
        rp = g.row_ptr[rb:re + 1]
        ci = g.col_idx[rp[0]:rp[-1]]
        col, halo, cnt = wl.halo_plan(g.n, bounds, rank, rp, ci)
        assert np.all(np.diff(halo) > 0) and np.all((halo < rb) | (halo >= re))
        assert cnt[rank] == 0 and cnt.sum() == len(halo)
        # requests grouped by owner (halo ids are sorted, partitions contiguous)
        offs = np.concatenate([[0], np.cumsum(cnt)])
        need = [halo[offs[p]:offs[p + 1]] for p in range(world)]
        all_need = [None] * world
        dist.all_gather_object(all_need, need)
        x = gg.vectors(g.n, 2, 5)  # the same seeded vector on every rank
        x_loc = x[rb:re]
        send = [x_loc[all_need[p][rank] - rb] if p != rank else None for p in range(world)]
        all_send = [None] * world
        dist.all_gather_object(all_send, send)
        x_halo = np.concatenate([all_send[p][rank] for p in range(world) if p != rank] +
                                [np.zeros((0, 2))])
        x_ext = np.vstack([x_loc, x_halo])
        y_loc = np.zeros_like(x_loc)
        lrp = rp - rp[0]
        for r in range(re - rb):
            y_loc[r] = x_ext[col[lrp[r]:lrp[r + 1]]].sum(axis=0)
        # Gram partials -> allreduce (gloo) == global inner products
        part = torch.from_numpy((y_loc * x_loc).sum(axis=0).copy())
        dist.all_reduce(part)
        ys = [None] * world
        dist.all_gather_object(ys, y_loc)
        if rank == 0:
            A = g.dense()
            y = np.vstack(ys)
            qout.put((float(np.max(np.abs(y - A @ x))), float(np.max(np.abs(part.numpy() - ((A @ x) * x).sum(0))))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partition_halo_exchange_spmv(world):
    from paper_2601_11338_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    err_y, err_dot = q.get(timeout=10)
    assert err_y < 1e-12           # the plan/exchange reproduces A x (summation order differs)
    assert err_dot < 1e-9
