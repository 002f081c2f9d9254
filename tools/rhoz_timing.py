import time, numpy as np, torch, sys
sys.path.insert(0, ".")
import graphgen as gg
from graphgen import configs
import paper_2601_11338_b200 as wl
cfg = configs.get("c4"); g = cfg["make"]()
op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.0], f=("series", [0.0, 1.0]), krylov_dim=2)
for i in range(6):
    torch.cuda.synchronize(); t = time.perf_counter()
    r = op.spectral_radius_z(0, k=60)
    torch.cuda.synchronize(); print("rhoz", r, round((time.perf_counter() - t) * 1e3, 1), "ms", flush=True)
H = np.triu(np.random.default_rng(0).standard_normal((61, 61)), -1)
t = time.perf_counter(); wl.hessenberg_eigvals(H); print("host QR 61x61", (time.perf_counter() - t) * 1e3, "ms")
