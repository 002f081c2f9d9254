"""Probe: do two independent Krylov actions on two CUDA streams overlap (latency-bound SpMM of one with
the bandwidth-bound basis passes of the other)?  C4 theta sweep split into two operators."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as gg  # noqa: E402
from graphgen import configs  # noqa: E402
import paper_2601_11338_b200 as wl  # noqa: E402

cfg = configs.get("c4")
g = cfg["make"]()
th = cfg["thetas"]
split = int(sys.argv[1]) if len(sys.argv) > 1 else 6
beta = 1.0 / 3372.2
ops = [wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=th[:split], f=("exp", beta)),
       wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=th[split:], f=("exp", beta))]
full = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=th, f=("exp", beta))
V = torch.from_numpy(gg.vectors(g.n, 1, 103)).cuda()
wss = [op.workspace(1) for op in ops]
wsf = full.workspace(1)
outs = [torch.empty((g.n, op.n_theta), dtype=torch.float64, device="cuda") for op in ops]
outf = torch.empty((g.n, full.n_theta), dtype=torch.float64, device="cuda")
streams = [torch.cuda.Stream(), torch.cuda.Stream()]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def one():
    full.apply(V, out=outf, ws=wsf)


def seq():
    for op, o, w in zip(ops, outs, wss):
        op.apply(V, out=o, ws=w)


def conc():
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for op, o, w, s in zip(ops, outs, wss, streams):
        with torch.cuda.stream(s):
            op.apply(V, out=o, ws=w, stream=s)
    for s in streams:
        cur.wait_stream(s)


print("single 11-column action   ms", round(timed(one), 1))
print(f"two actions ({split}+{len(th)-split}) sequential ms", round(timed(seq), 1))
print(f"two actions concurrent    ms", round(timed(conc), 1))
