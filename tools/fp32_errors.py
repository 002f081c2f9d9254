"""Print the fp32 mode's relative errors vs the series oracle (tests/test_gpu_fp32.py cases, mid-size)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import graphgen as gg  # noqa: E402
import paper_2601_11338_b200 as wl  # noqa: E402
from oracle import coeffs as C  # noqa: E402
from oracle import series as S  # noqa: E402


def relerr(got, ref):
    den = np.linalg.norm(ref, axis=0)
    den[den == 0] = 1.0
    return np.linalg.norm(got - ref, axis=0) / den


for g in (gg.rmat(14, 12000, 150000, seed=21, perm_seed=22), gg.barabasi_albert(20000, 5, 31),
          gg.grid_lcc(150, 149, 0.3, 41), gg.rmat(17, 100000, 1500000, seed=5, perm_seed=6)):
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 5, 77)
    thetas = [0.0, 0.5, 1.0]
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param), fp32=1)
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    op.close()
    errs = [relerr(got[:, 5 * i:5 * i + 5], S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() for i, th in enumerate(thetas)]
    print(g.name, g.n, " ".join(f"theta={th}: {e:.2e}" for th, e in zip(thetas, errs)))
