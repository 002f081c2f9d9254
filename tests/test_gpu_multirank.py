"""GPU parity of the row-partitioned (multi-rank) path on ONE device: the loopback transport.

P ranks live in this process (one host thread and one CUDA stream each, wl_comm_create_loopback).
They run the multi-rank code path itself: nnz-balanced rows (wl_partition), the halo plan with the
relabelled send ids, `pack_rows`, the HALO instantiations of the SpMM kernels, the grouped halo
exchange (device copies instead of NCCL send/recv) and the allreduce of every Gram pass (a
fixed-order device sum instead of ncclAllReduce), so H and every coefficient are replicated on all
ranks ("transparently on one or more GPU accelerators").  Results, gathered
row block by row block, are compared with the CPU oracle (relative L2 per column <= 1e-10) and with
the same operator on one rank (<= 1e-13: the only differences are summation orders).
"""
import numpy as np
import pytest

import graphgen as gg
from oracle import coeffs as C
from oracle import dense as D
from oracle import series as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-10
TOL_P1 = 1e-13


@pytest.fixture(scope="module")
def wl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_11338_b200 as wl
    from paper_2601_11338_b200 import build
    build.build()
    wl.load()
    return wl


def relerr(got, ref):
    got, ref = np.atleast_2d(got.T).T, np.atleast_2d(ref.T).T
    den = np.linalg.norm(ref, axis=0)
    den[den == 0] = 1.0
    return np.linalg.norm(got - ref, axis=0) / den


def _rows(g, bounds, r):
    rb, re = int(bounds[r]), int(bounds[r + 1])
    rp = g.row_ptr[rb:re + 1]
    return rb, re, rp, g.col_idx[rp[0]:rp[-1]]


def run_ranks(wl, g, P, body, bounds=None, **opkw):
    """Build the P-rank operator of g and run body(op, rb, re, stream) on every rank; returns the
    per-rank results and the ranks' halo sizes."""
    bounds = wl.partition(g.row_ptr, P) if bounds is None else np.asarray(bounds, dtype=np.int64)

    def rank_fn(r, comm, stream):
        rb, re, rp, ci = _rows(g, bounds, r)
        op = wl.Operator(g.n, rp, ci, row_range=(rb, re), comm=comm, stream=stream, **opkw)
        try:
            out = body(op, rb, re, stream)
            stream.synchronize()
            return out, op.n_halo
        finally:
            op.close()

    res = wl.run_loopback(P, rank_fn, timeout=300.0)
    return [x[0] for x in res], [x[1] for x in res]


GRAPHS = {
    "rmat": lambda: gg.rmat(13, 6000, 60000, seed=21, perm_seed=22),     # hubs + ~35% isolated rows
    "ba": lambda: gg.barabasi_albert(8000, 5, 31),
    "road": lambda: gg.grid_lcc(90, 89, 0.3, 41),
}


@pytest.mark.parametrize("overlap", [1, 0])
@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_loopback_apply_vs_oracle_and_one_rank(wl, name, P, overlap):
    """wl_apply and t_θ on P ranks for θ ∈ {1, 0.5, 0} (one batched sweep) against the series oracle
    and against P = 1; every rank with a halo exercises the exchange.  overlap = 1: the A_loc SpMM runs
    while the halo is exchanged on the comm stream and the A_halo SpMM accumulates after it."""
    g = GRAPHS[name]()
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    thetas = [1.0, 0.5, 0.0]
    b = 2
    V = gg.vectors(g.n, b, 77)
    kw = dict(thetas=thetas, f=("exp", f.param))
    op1 = wl.Operator(g.n, g.row_ptr, g.col_idx, **kw)
    ref1 = op1.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    t1 = op1.diag_shift().cpu().numpy()
    op1.close()

    def body(op, rb, re, stream):
        Vl = torch.from_numpy(V[rb:re].copy()).cuda()
        LV = op.apply(Vl, stream=stream)
        t = op.diag_shift(stream=stream)
        stream.synchronize()
        return LV.cpu().numpy(), t.cpu().numpy()

    res, halos = run_ranks(wl, g, P, body, halo_overlap=overlap, **kw)
    assert sum(h > 0 for h in halos) >= 2, halos
    LV = np.vstack([r[0] for r in res])
    t = np.vstack([r[1] for r in res])
    assert relerr(LV, ref1).max() < TOL_P1
    assert relerr(t, t1).max() < TOL_P1
    for i, th in enumerate(thetas):
        ref = S.laplacian_apply(g, 1.0 - th, f, V, rA)
        assert relerr(LV[:, i * b:(i + 1) * b], ref).max() < TOL, th
        assert relerr(t[:, i], S.total_communicability(g, 1.0 - th, f, rA)).max() < TOL, th


@pytest.mark.parametrize("relabel", [0, 1])
@pytest.mark.parametrize("reorth", [1, 2])
def test_loopback_orthogonalisation_and_relabel(wl, relabel, reorth):
    """DCGS2 and TOAR, relabelling on and off (the relabelled send ids of the halo plan)."""
    g = gg.rmat(12, 3000, 30000, seed=5, perm_seed=6)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 3, 9)
    kw = dict(thetas=[0.25, 0.75], f=("exp", f.param), relabel=relabel, reorth=reorth)

    def body(op, rb, re, stream):
        return op.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream).cpu().numpy()

    LV = np.vstack(run_ranks(wl, g, 3, body, **kw)[0])
    for i, th in enumerate([0.25, 0.75]):
        assert relerr(LV[:, i * 3:(i + 1) * 3], S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() < TOL


def test_loopback_diffusion(wl):
    """a9 exp(-τ𝕃)x0 on 3 ranks vs the dense eigendecomposition and vs one rank."""
    g = gg.grid_lcc(30, 30, 0.3, 5)
    A = D.adjacency(g)
    rA = D.rho_A(A)
    ts = np.linspace(0, 100, 19)
    x0 = np.zeros(g.n)
    x0[g.n // 2] = 1.0
    kw = dict(thetas=[0.0], f=("exp", 1.0 / rA))
    op1 = wl.Operator(g.n, g.row_ptr, g.col_idx, **kw)
    X1 = op1.diffuse(torch.from_numpy(x0).cuda(), ts, k_out=80).cpu().numpy()
    op1.close()

    def body(op, rb, re, stream):
        return op.diffuse(torch.from_numpy(x0[rb:re].copy()).cuda(), ts, k_out=80, stream=stream).cpu().numpy()

    X = np.vstack(run_ranks(wl, g, 3, body, **kw)[0])
    ref = D.diffusion(D.laplacian(A, 1.0, C.exp(1.0 / rA)), x0, ts)
    assert relerr(X, ref).max() < TOL
    assert relerr(X, X1).max() < 1e-12
    assert np.max(np.abs(X.sum(0) - 1.0)) < 1e-10


@pytest.mark.parametrize("overlap", [1, 0])
def test_loopback_cg_resolvent(wl, overlap):
    """NEXT-1: the resolvent by PCG on 𝒜_θ(α) on 4 ranks (halo before each SpMM, allreduce per scalar)."""
    g = gg.barabasi_albert(3000, 4, 2)
    A = D.adjacency(g)
    alpha = 0.5 / D.rho_A(A)
    V = gg.vectors(g.n, 2, 4)
    kw = dict(thetas=[0.0, 0.5], f=("resolvent", alpha), solver="cg", cg_tol=1e-13, halo_overlap=overlap)

    def body(op, rb, re, stream):
        return op.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream).cpu().numpy()

    LV = np.vstack(run_ranks(wl, g, 4, body, **kw)[0])
    for i, th in enumerate([0.0, 0.5]):
        ref = D.walk_laplacian(D.phi_resolvent_closed(A, 1.0 - th, alpha)) @ V
        assert relerr(LV[:, 2 * i:2 * i + 2], ref).max() < 1e-10


def test_loopback_spectral_radius_z(wl):
    g = gg.karate()
    A = D.adjacency(g)

    def body(op, rb, re, stream):
        return op.spectral_radius_z(0, k=60, stream=stream)

    rhos, _ = run_ranks(wl, g, 2, body, variant="nbt", f=("exp", 0.1))
    assert rhos[0] == rhos[1]                         # replicated Hessenberg matrix
    assert abs(rhos[0] - D.rho_Z(A, 1.0)) < 1e-9 * D.rho_Z(A, 1.0)


def test_loopback_empty_rank(wl):
    """A rank with no rows (ADVICE: launches with grid 0) still joins every collective."""
    g = gg.barabasi_albert(2000, 3, 8)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 1, 3)
    ts = [0.5, 2.0]
    bounds = [0, 0, 700, g.n]                          # rank 0 owns nothing
    kw = dict(thetas=[0.5], f=("exp", f.param))

    def body(op, rb, re, stream):
        LV = op.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream)
        X = op.diffuse(torch.from_numpy(np.ascontiguousarray(V[rb:re, 0])).cuda(), ts, k_out=40, stream=stream)
        return LV.cpu().numpy(), X.cpu().numpy()

    res, halos = run_ranks(wl, g, 3, body, bounds=bounds, **kw)
    LV = np.vstack([r[0] for r in res])
    X = np.vstack([r[1] for r in res])
    assert res[0][0].shape[0] == 0 and halos[0] == 0
    assert relerr(LV, S.laplacian_apply(g, 0.5, f, V, rA)).max() < TOL
    ref = D.diffusion(D.laplacian(D.adjacency(g), 0.5, f), V[:, 0], ts)
    assert relerr(X, ref).max() < TOL
    op1 = wl.Operator(g.n, g.row_ptr, g.col_idx, **kw)
    X1 = op1.diffuse(torch.from_numpy(np.ascontiguousarray(V[:, 0])).cuda(), ts, k_out=40).cpu().numpy()
    op1.close()
    assert relerr(X, X1).max() < 1e-12


def test_loopback_lanczos_adaptive_and_rational_trace(wl):
    """The round-2 paths across ranks: the μ = 0 Lanczos batches (per-column scalars allreduced), the adaptive
    Krylov stop (every rank takes the same decision from the replicated H), and the rational XNysTrace-exp (MINRES
    scalars allreduced, the Cholesky-QR and Rayleigh-quotient Gram blocks allreduced) — each against P = 1."""
    g = gg.barabasi_albert(3000, 4, 2)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 2, 4)
    Om = gg.vectors(g.n, 4, 9)
    ts = np.linspace(0.0, 5.0, 7)
    poles = np.array([np.inf, -2.5, -1.0 + 3.0j])
    kw_walk = dict(variant="walk", f=("exp", f.param))
    kw_ad = dict(thetas=[0.0, 0.5], f=("exp", f.param), krylov_tol=1e-13, krylov_adaptive=1)

    def one_rank():
        o = wl.Operator(g.n, g.row_ptr, g.col_idx, **kw_walk)
        a = o.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        o.close()
        o = wl.Operator(g.n, g.row_ptr, g.col_idx, **kw_ad)
        b = o.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        p, e, _ = o.xnystrace_exp_rational(torch.from_numpy(Om).cuda(), ts, poles=poles, inner_tol=1e-13)
        o.close()
        return a, b, p

    a1, b1, p1 = one_rank()
    bounds = wl.partition(g.row_ptr, 3)

    def rank_fn(r, comm, stream):
        rb, re = int(bounds[r]), int(bounds[r + 1])
        rp = g.row_ptr[rb:re + 1]
        ci = g.col_idx[rp[0]:rp[-1]]
        o = wl.Operator(g.n, rp, ci, row_range=(rb, re), comm=comm, stream=stream, **kw_walk)
        a = o.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream).cpu().numpy()
        o.close()
        o = wl.Operator(g.n, rp, ci, row_range=(rb, re), comm=comm, stream=stream, **kw_ad)
        b = o.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream).cpu().numpy()
        p, e, _ = o.xnystrace_exp_rational(torch.from_numpy(Om[rb:re].copy()).cuda(), ts, poles=poles,
                                           inner_tol=1e-13, stream=stream)
        o.close()
        return a, b, p

    res = wl.run_loopback(3, rank_fn, timeout=300.0)
    assert relerr(np.vstack([r[0] for r in res]), a1).max() < TOL_P1
    assert relerr(np.vstack([r[1] for r in res]), b1).max() < TOL_P1
    for r in res:
        assert np.max(np.abs(r[2] - p1) / np.abs(p1)) < 1e-11
    assert relerr(a1, S.laplacian_apply(g, 0.0, f, V, rA)).max() < TOL
