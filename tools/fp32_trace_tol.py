"""fp32 / fp64 rational XNysTrace (Fig. 7 shape, mid-size road grid) vs the oracle's exact solves, per inner tol."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import graphgen as gg  # noqa: E402
import paper_2601_11338_b200 as wl  # noqa: E402
from oracle import coeffs as C  # noqa: E402
from oracle import dense as D  # noqa: E402
from oracle import trace as T  # noqa: E402

g = gg.grid_lcc(60, 60, 0.3, 2002)
A = D.adjacency(g)
rA = D.rho_A(A)
Lap = D.laplacian(A, 1.0, C.exp(1.0 / rA))
ts = np.linspace(0.0, 100.0, 90)
Om = gg.vectors(g.n, 30, 2026)
op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.0], f=("exp", 1.0 / rA))
poles = wl.aaa_exp_poles(max(ts) * op.laplacian_bound(0))
op.close()
po, eo = T.xnystrace_exp_rational(Lap, Om, poles, ts)
for fp32 in (0, 1):
    for tol in (1e-6, 1e-7, 1e-8, 1e-9, 1e-10, 1e-12):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.0], f=("exp", 1.0 / rA), fp32=fp32)
        try:
            p, e, info = op.xnystrace_exp_rational(torch.from_numpy(Om).cuda(), ts, poles=poles, inner_tol=tol,
                                                   inner_maxit=3000)
            print(f"fp32={fp32} tol={tol:g}: max rel err {np.max(np.abs(p - po) / np.abs(po)):.2e} iters {info['inner_iters']}",
                  flush=True)
        except Exception as ex:
            print(f"fp32={fp32} tol={tol:g}: {ex}", flush=True)
        op.close()
