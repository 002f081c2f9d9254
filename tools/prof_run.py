"""Small driver for ncu / timing experiments: build a config's operator and run a few actions.
usage: python tools/prof_run.py [config] [krylov_dim] [steps] [b]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as gg  # noqa: E402
from graphgen import configs  # noqa: E402
import paper_2601_11338_b200 as wl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
b = int(sys.argv[4]) if len(sys.argv) > 4 else 0
cfg = configs.get(name)
t0 = time.time()
g = cfg["make"]()
print(f"graph {g.n} {g.nnz} in {time.time()-t0:.1f}s", flush=True)
op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=cfg["thetas"], f=("exp", 1.0 / 3000.0), krylov_dim=K)
b = b or cfg["b"]
V = torch.from_numpy(gg.vectors(g.n, b, 1)).cuda()
out = torch.empty((g.n, op.n_theta * b), dtype=torch.float64, device="cuda")
ws = op.workspace(b)
torch.cuda.synchronize()
for i in range(steps):
    t1 = time.time()
    op.apply(V, out=out, ws=ws)
    torch.cuda.synchronize()
    print(f"step {i}: {1e3*(time.time()-t1):.1f} ms", flush=True)
