"""Small run through every kernel family for compute-sanitizer (racecheck / synccheck / memcheck):
the bulk-copy ring passes (TOAR dots/update, DCGS2 dots/update), the hub-row chunk tickets of the SpMM
(a 9000-neighbour hub: three 4096-nonzero chunks), the batched small rows, the 32-byte lane
gathers (B = 11 over a padded block), CG, the outer diffusion Arnoldi, and the loopback halo exchange.
Checks the results against the oracle so a silent corruption also fails.
    compute-sanitizer --tool racecheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
import paper_2601_11338_b200 as wl  # noqa: E402
from oracle import coeffs as C  # noqa: E402
from oracle import series as S  # noqa: E402


def relerr(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=0) / np.linalg.norm(b, axis=0)))


def main():
    wl.load()
    # a hub of 3000 leaves (2 chunks of 2048 nonzeros) attached to a small R-MAT
    r = gg.rmat(10, 900, 4000, seed=3, perm_seed=4)
    edges = [(int(i), int(j)) for i in range(r.n) for j in r.col_idx[r.row_ptr[i]:r.row_ptr[i + 1]] if i < j]
    n = r.n + 9001
    edges += [(r.n, r.n + 1 + k) for k in range(9000)] + [(0, r.n)]
    g = gg.from_edges(n, edges)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    thetas = [round(0.1 * i, 1) for i in range(11)]
    V = gg.vectors(n, 1, 5)
    worst = 0.0
    for reorth in (2, 1):
        op = wl.Operator(n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param), reorth=reorth, krylov_dim=12)
        LV = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        for i in (0, 5, 10):
            worst = max(worst, relerr(LV[:, i:i + 1], S.laplacian_apply(g, 1.0 - thetas[i], f, V, rA)))
        x0 = np.zeros(n)
        x0[0] = 1.0
        X = op.diffuse(torch.from_numpy(x0).cuda(), [0.5, 1.0], k_out=8, theta_index=5).cpu().numpy()
        assert np.all(np.isfinite(X))
        op.close()
    alpha = 0.5 / rA
    op = wl.Operator(n, g.row_ptr, g.col_idx, thetas=[0.0, 1.0], f=("resolvent", alpha), solver="cg", cg_tol=1e-12)
    op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    op.close()
    # two loopback ranks: pack_rows, HALO gathers, the A_loc / A_halo split and the comm stream
    bounds = wl.partition(g.row_ptr, 2)

    def rank_fn(rk, comm, stream):
        rb, re = int(bounds[rk]), int(bounds[rk + 1])
        rp = g.row_ptr[rb:re + 1]
        o = wl.Operator(n, rp, g.col_idx[rp[0]:rp[-1]], row_range=(rb, re), comm=comm, stream=stream,
                        thetas=[0.0, 0.5], f=("exp", f.param), krylov_dim=8)
        out = o.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream).cpu().numpy()
        o.close()
        return out

    LV2 = np.vstack(wl.run_loopback(2, rank_fn))
    o1 = wl.Operator(n, g.row_ptr, g.col_idx, thetas=[0.0, 0.5], f=("exp", f.param), krylov_dim=8)
    LV1 = o1.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    o1.close()
    worst = max(worst, relerr(LV2, LV1))
    torch.cuda.synchronize()
    print(f"sanitize_case: ok, max rel err {worst:.2e}")
    assert worst < 1e-9


if __name__ == "__main__":
    main()
