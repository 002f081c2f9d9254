"""GPU parity of the fp32 mode (wl_opts.fp32) vs the CPU oracle.

The north star fixes the bar: relative L2 error per column <= 1e-4 "for any fp32 mode" (BASELINE.json).
In this mode the n-vectors of each TOAR batch (the basis U, the SpMM's gathered operand and its output)
are stored in float; every sum (SpMM rows, dot products, basis updates, combine) and the projected work
stay double, inputs/outputs are double and t_θ (create time) is computed in double (so it keeps the fp64
bar).  Cases: the multi-tile graphs of test_gpu_parity for θ ∈ {1, 0.5, 0} (θ = 0: |γ| = d - 1 against
ρ(A), the hardest column) at b ∈ {1, 5}; batch widths B = 1..17 over hub chunks (the 8-float 32-byte
lanes with 1-3 lanes per row, and the scalar-lane B = 1 path); two Krylov batches; the adaptive stop; the
diffusion inner actions; the row-partitioned path on loopback ranks; the options it rejects.
"""
import numpy as np
import pytest

import graphgen as gg
from oracle import coeffs as C
from oracle import dense as D
from oracle import series as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL32 = 1e-4   # north_star: fp32 mode
TOL64 = 1e-10  # t_θ stays double


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


@pytest.mark.parametrize("theta", [1.0, 0.5, 0.0])
def test_fp32_multi_tile_graphs_vs_series(wl, theta):
    graphs = [gg.rmat(14, 12000, 150000, seed=21, perm_seed=22),
              gg.barabasi_albert(20000, 5, 31),
              gg.grid_lcc(150, 149, 0.3, 41)]
    for g in graphs:
        rA = S.rho_A(g)
        f = C.exp(1.0 / rA)
        for b in (1, 5):
            V = gg.vectors(g.n, b, 77)
            op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[theta], f=("exp", f.param), fp32=1)
            got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
            ref = S.laplacian_apply(g, 1.0 - theta, f, V, rA)
            err = relerr(got, ref).max()
            assert err < TOL32, (g.name, b, err)
            assert err > 1e-13, "fp32 storage must be visible in the error (is the mode on?)"
            t = op.diag_shift().cpu().numpy()[:, 0]
            assert relerr(t, S.total_communicability(g, 1.0 - theta, f, rA)).max() < TOL64
            op.close()


@pytest.mark.parametrize("B", [1, 2, 4, 8, 11, 16, 17])
def test_fp32_batch_widths_over_hub_chunks(wl, B):
    """B columns of one θ (b = B): 8-float lanes with W = ceil(B/8) lanes per gathered row (B = 2..17), the
    scalar B = 1 path; rows longer than a hub chunk (4096) reduced across warps."""
    rng = np.random.default_rng(5)
    n = 20000
    edges = set()
    for hub, deg in ((0, 10000), (1, 4097), (2, 8193), (3, 700), (4, 2049)):
        for v in rng.choice(np.arange(5, n), size=deg, replace=False):
            edges.add((min(hub, int(v)), max(hub, int(v))))
    for _ in range(20000):
        a, c = rng.integers(5, n, size=2)
        if a != c:
            edges.add((min(a, c), max(a, c)))
    g = gg.from_edges(n, sorted(edges), "hubs")
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, B, 8)
    for th in (0.0, 0.6):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[th], f=("exp", f.param), fp32=1)
        got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        assert relerr(got, S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() < TOL32, (B, th)
        op.close()


def test_fp32_theta_sweep_two_batches_and_functions(wl):
    """11 θ x b = 3 = 33 columns (two Krylov batches); the resolvent and a series walk function too."""
    g = gg.rmat(12, 3000, 30000, seed=3, perm_seed=4)
    rA = S.rho_A(g)
    thetas = list(np.linspace(0.0, 1.0, 11))
    V = gg.vectors(g.n, 3, 8)
    for f, spec in ((C.exp(1.0 / rA), ("exp", 1.0 / rA)),
                    (C.resolvent(0.5 / rA), ("resolvent", 0.5 / rA)),
                    (C.series([1.0, 0.5, 0.25, 0.125]), ("series", [1.0, 0.5, 0.25, 0.125]))):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=spec, fp32=1)
        got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        for i, th in enumerate(thetas):
            ref = S.laplacian_apply(g, 1.0 - th, f, V, rA)
            assert relerr(got[:, 3 * i:3 * i + 3], ref).max() < TOL32, (spec[0], th)
        op.close()


def test_fp32_adaptive_and_diffusion(wl):
    g = gg.grid_lcc(30, 30, 0.3, 5)
    A = D.adjacency(g)
    rA = D.rho_A(A)
    ts = np.linspace(0, 100, 19)
    x0 = np.zeros(g.n)
    x0[g.n // 2] = 1.0
    for th in (1.0, 0.0):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[th], f=("exp", 1.0 / rA), fp32=1)
        X = op.diffuse(torch.from_numpy(x0).cuda(), ts, k_out=80).cpu().numpy()
        ref = D.diffusion(D.laplacian(A, 1.0 - th, C.exp(1.0 / rA)), x0, ts)
        assert relerr(X, ref).max() < TOL32, th
        op.close()
    g = gg.rmat(14, 12000, 150000, seed=21, perm_seed=22)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 2, 7)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.0, 0.5], f=("exp", f.param), krylov_dim=40,
                     krylov_tol=1e-8, krylov_adaptive=1, fp32=1)
    ws = op.workspace(2)
    LV = op.apply(torch.from_numpy(V).cuda(), ws=ws).cpu().numpy()
    _, steps, batches = ws.stats()
    op.close()
    assert steps / batches < 40
    for i, th in enumerate((0.0, 0.5)):
        assert relerr(LV[:, 2 * i:2 * i + 2], S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() < TOL32, th


def test_fp32_loopback_ranks(wl):
    """The row-partitioned path with float halo rows (pack, exchange, HALO kernels) on 3 loopback ranks, with
    and without the A_loc / A_halo overlap, vs the oracle and vs the fp32 operator on one rank."""
    g = gg.rmat(13, 6000, 60000, seed=21, perm_seed=22)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    thetas = [1.0, 0.5, 0.0]
    b = 2
    V = gg.vectors(g.n, b, 77)
    kw = dict(thetas=thetas, f=("exp", f.param), fp32=1)
    op1 = wl.Operator(g.n, g.row_ptr, g.col_idx, **kw)
    ref1 = op1.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    op1.close()
    bounds = wl.partition(g.row_ptr, 3)
    for overlap in (1, 0):
        def rank_fn(r, comm, stream):
            rb, re = int(bounds[r]), int(bounds[r + 1])
            rp = g.row_ptr[rb:re + 1]
            op = wl.Operator(g.n, rp, g.col_idx[rp[0]:rp[-1]], row_range=(rb, re), comm=comm, stream=stream,
                             halo_overlap=overlap, **kw)
            try:
                out = op.apply(torch.from_numpy(V[rb:re].copy()).cuda(), stream=stream)
                stream.synchronize()
                return out.cpu().numpy(), op.n_halo
            finally:
                op.close()

        res = wl.run_loopback(3, rank_fn, timeout=300.0)
        assert sum(h > 0 for _, h in res) >= 2
        LV = np.vstack([x[0] for x in res])
        assert relerr(LV, ref1).max() < 1e-5, overlap   # same storage, other summation orders
        for i, th in enumerate(thetas):
            ref = S.laplacian_apply(g, 1.0 - th, f, V, rA)
            assert relerr(LV[:, i * b:(i + 1) * b], ref).max() < TOL32, (overlap, th)


def test_fp32_rejected_combinations(wl):
    g = gg.karate()
    for kw in (dict(reorth=1), dict(reorth=0), dict(solver="cg", f=("resolvent", 0.05))):
        args = dict(thetas=[0.5], f=("exp", 0.1), fp32=1)
        args.update(kw)
        with pytest.raises(Exception):
            wl.Operator(g.n, g.row_ptr, g.col_idx, **args)


@pytest.mark.slow
def test_fp32_full_c4_theta_sweep_vs_series(wl):
    """C4 at full size (R-MAT n=1e7, nnz=4e8, 11 θ, b = 1, k = 30) in the fp32 mode — the bench's --fp32
    line — vs the series oracle for θ ∈ {0, 0.5, 1}; t_θ at the fp64 bar."""
    from graphgen import configs
    cfg = configs.get("c4")
    g = cfg["make"]()
    A = S.csr(g)
    rho = S.rho_A(g, tol=1e-10)
    beta = 1.0 / rho
    V = gg.vectors(g.n, 1, cfg["vec_seed"])
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=cfg["thetas"], f=("exp", beta), krylov_dim=30, fp32=1)
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    t_gpu = op.diag_shift().cpu().numpy()
    op.close()
    f = C.exp(beta)
    ones_v = np.stack([np.ones(g.n), V[:, 0]], axis=1)
    for th in (0.0, 0.5, 1.0):
        i = cfg["thetas"].index(th)
        phi = S.phi_apply(g, 1.0 - th, f, ones_v, rho * 1.001, A=A)
        ref = phi[:, 0] * V[:, 0] - phi[:, 1]
        assert relerr(t_gpu[:, i], phi[:, 0]).max() < TOL64, th
        assert relerr(got[:, i], ref).max() < TOL32, th


def _rational_fp32(wl, g, theta, M, ts, seed, poles=None, inner_tol=1e-7):
    from oracle import trace as T
    A = D.adjacency(g)
    rA = D.rho_A(A)
    Lap = D.laplacian(A, 1.0 - theta, C.exp(1.0 / rA))
    Om = gg.vectors(g.n, M, seed)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[theta], f=("exp", 1.0 / rA), fp32=1)
    if poles is None:
        poles = wl.aaa_exp_poles(max(ts) * op.laplacian_bound(0))
    p, e, info = op.xnystrace_exp_rational(torch.from_numpy(Om).cuda(), ts, poles=poles, inner_tol=inner_tol,
                                           inner_maxit=2000)
    op.close()
    po, eo = T.xnystrace_exp_rational(Lap, Om, poles, ts)
    return p, e, po, eo


def test_fp32_rational_trace_every_pole_kind(wl):
    """NEXT-2 (Alg. 1, rational) with fp32 inner actions (MINRES shifted solves to 1e-7 on float-stored Krylov
    batches): ∞, a real pole and a conjugate pair on a BA graph, vs the oracle's dense solves, p̂ at the 1e-4 bar."""
    g = gg.barabasi_albert(1201, 3, 5)
    ts = np.linspace(0.0, 4.0, 9)
    p, e, po, eo = _rational_fp32(wl, g, 0.0, 5, ts, 3, poles=np.array([np.inf, -2.5, -1.0 + 3.0j, 0.5 + 6.0j]))
    assert np.max(np.abs(p - po) / np.abs(po)) < TOL32


@pytest.mark.slow
def test_fp32_rational_midsize_road_fig7_shape(wl):
    """The Fig. 7 shape (road-like grid, NBT, M = 30, 90 t in [0, 100], the library's AAA poles) with fp32 inner
    actions, vs the oracle's exact shifted solves: p̂ at the 1e-4 bar.  MINRES to 1e-10: with the paper's 1e-6
     the inexact solves alone move p̂(100) by 2e-3 relative in fp64 and fp32 alike (tools/fp32_trace_tol.py:
    1e-7 -> 4e-4, 1e-8 -> 7e-6, 1e-10 -> 1.3e-7 (fp32) / 1.5e-7 (fp64))."""
    g = gg.grid_lcc(60, 60, 0.3, 2002)
    p, e, po, eo = _rational_fp32(wl, g, 0.0, 30, np.linspace(0.0, 100.0, 90), 2026, inner_tol=1e-10)
    assert np.max(np.abs(p - po) / np.abs(po)) < TOL32


def test_fp32_fuzz_small_graphs(wl):
    """Randomised small cases (n <= 30, random density incl. isolated vertices, θ incl. 1 (Lanczos batches), walk
    function, b; k = 64 >= 2n exhausts the Krylov space, so the only error is the float storage) in the fp32 mode
    vs the dense oracle at 1e-4."""
    rng = np.random.default_rng(4321)
    for case in range(25):
        n = int(rng.integers(2, 31))
        p = float(rng.uniform(0.05, 0.6))
        e = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        if not e:
            e = [(0, 1)]
        g = gg.from_edges(n, e, f"fuzz32_{case}")
        A = D.adjacency(g)
        rA = max(D.rho_A(A), 1.0)
        kind = ("exp", "resolvent", "series")[case % 3]
        if kind == "exp":
            f, fo = ("exp", 1.0 / rA), C.exp(1.0 / rA)
        elif kind == "resolvent":
            a = float(rng.uniform(0.05, 0.8)) / rA
            f, fo = ("resolvent", a), C.resolvent(a)
        else:
            cs = list(rng.uniform(0.0, 1.0, size=int(rng.integers(2, 7))))
            f, fo = ("series", cs), C.series(cs)
        thetas = [1.0] if case % 4 == 0 else list(np.round(rng.uniform(0, 1, size=int(rng.integers(1, 4))), 3))
        b = int(rng.integers(1, 4))
        V = gg.vectors(n, b, 200 + case)
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=f, krylov_dim=64, fp32=1)
        got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        for i, th in enumerate(thetas):
            ref = D.walk_laplacian(D.phi(A, 1.0 - th, fo)) @ V
            err = relerr(got[:, i * b:(i + 1) * b], ref).max()
            assert err < TOL32, (case, n, kind, th, b, err)
        op.close()
