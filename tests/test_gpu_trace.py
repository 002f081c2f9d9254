"""GPU parity of XNysTrace-exp (Alg. 1 with poles at ∞) vs oracle/trace.py.

Both sides take the same seeded Gaussian probes Ω (graphgen.vectors) and the same k; the oracle
runs block Arnoldi and the estimator on the dense 𝕃 from oracle/dense.py, the GPU path runs k
batched Laplacian actions through the C ABI (wl_xnystrace_exp).  Rounding differs (Gram–Schmidt
order, Jacobi vs scaling-and-squaring expm), so the estimates agree to 1e-8 relative — the
estimator's leave-one-out Gram matrices have condition numbers up to ~1/ν ≈ 1e12 at large t —
far below its own statistical error (ê, 1e-3..1e-1 here).
"""
import numpy as np
import pytest

import graphgen as gg
from oracle import coeffs as C
from oracle import dense as D
from oracle import trace as T

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def wl():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2601_11338_b200 as wl
    from paper_2601_11338_b200 import build
    build.build()
    wl.load()
    return wl


def _case(wl, g, thetas, f, ti, M, k, ts, seed, **kw):
    A = D.adjacency(g)
    fo = {"exp": C.exp, "resolvent": C.resolvent}[f[0]](f[1])
    Lap = D.laplacian(A, 1.0 - thetas[ti], fo)
    Om = gg.vectors(g.n, M, seed)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=f, **kw)
    p, e = op.xnystrace_exp(torch.from_numpy(Om).cuda(), ts, k, theta_index=ti)
    op.close()
    po, eo = T.xnystrace_exp(Lap, Om, k, ts)
    return p, e, po, eo


# karate's 𝕃 has a 4-fold eigenvalue, so its block Krylov spaces stop growing before kM = 34: kM ≤ 24
@pytest.mark.parametrize("M,k", [(1, 6), (4, 6), (8, 3)])
def test_karate_exp_vs_oracle(wl, M, k):
    g = gg.karate()
    rA = D.rho_A(D.adjacency(g))
    ts = np.linspace(0.0, 10.0, 30)
    p, e, po, eo = _case(wl, g, [0.0, 0.5, 1.0], ("exp", 1.0 / rA), 1, M, k, ts, 7 + M)
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-8
    assert np.max(np.abs(e - eo)) < 1e-8 * np.max(np.abs(po)) + 1e-6 * np.max(eo)


def test_fig4b_shape_nbt_resolvent(wl):
    """Fig. 4(b) workload: 𝕃_1((1-αx)^{-1}) on karate, α = 1/(1+ρ(Z)), M = 3 (caption P:1260)."""
    g = gg.karate()
    alpha = 1.0 / (1.0 + D.rho_Z(D.adjacency(g), 1.0))
    ts = np.linspace(0.0, 10.0, 30)
    p, e, po, eo = _case(wl, g, [0.0], ("resolvent", alpha), 0, 3, 10, ts, 99, krylov_dim=64)  # θ = 0: NBT
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-8


def test_multi_tile_graph(wl):
    """A Barabási–Albert graph spanning many SpMM tiles and a ragged tail (n = 1201)."""
    g = gg.barabasi_albert(1201, 3, 5)
    rA = D.rho_A(D.adjacency(g))
    ts = np.linspace(0.0, 4.0, 9)
    p, e, po, eo = _case(wl, g, [0.7], ("exp", 1.0 / rA), 0, 6, 6, ts, 3)
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-8
    assert p[0] > 0 and np.all(e >= 0)


def test_argument_errors(wl):
    g = gg.karate()
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0], f=("exp", 0.1))
    Om = torch.from_numpy(gg.vectors(34, 4, 1)).cuda()
    with pytest.raises(Exception):
        op.xnystrace_exp(Om, [0.0, 1.0], 9)          # k*M = 36 > n = 34
    with pytest.raises(Exception):
        op.xnystrace_exp(Om, [-1.0], 2)              # negative time
    op.close()


def test_full_c3_fig7_shape(wl):
    """Full C3 (n ≈ 2e6 road-like grid, NBT θ = 0) in the Fig. 7 shape (M = 30, 90 t-points), as
    bench.py --trace runs it.  At t = 0, Y(0) = Ω/n exactly (exp(0) = I), so p̂(0), ê(0) depend only on Ω
    and the oracle's XNysTrace computes them at full size; the curve must decrease like (1/n)tr e^{-t𝕃}
    (every eigenvalue of 𝕃 is ≥ 0) within its error estimate, and stay above 1/n."""
    from graphgen import configs
    cfg = configs.get("c3")
    g = cfg["make"]()
    probe = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0], f=("series", [0.0, 1.0]), krylov_dim=2)
    rho = probe.spectral_radius(k=60)
    probe.close()
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.0], f=("exp", 1.0 / rho), krylov_dim=30)
    Om = gg.vectors(g.n, 30, 2026)
    ts = np.linspace(0.0, 10.0, 90)
    p, e = op.xnystrace_exp(torch.from_numpy(Om).cuda(), ts, 8)
    op.close()
    p0, e0 = T.xnystrace(Om / g.n, Om)
    assert abs(p[0] - p0) <= 1e-9 * abs(p0)
    assert abs(e[0] - e0) <= 1e-6 * e0
    assert np.all(np.diff(p) <= 3 * (e[1:] + e[:-1]))
    assert np.all(p > 1.0 / g.n)


@pytest.mark.slow
def test_midsize_road_full_curve_fig7_shape(wl):
    """The bench's launch configuration (M = 30 probes, k = 8 block steps, 90 t-points, NBT θ = 0 on a
    road-like grid) on a graph the dense oracle handles (n ≈ 2.5e3): the WHOLE curve p̂(t) and ê(t)
    against oracle/trace.py, not only t = 0."""
    g = gg.grid_lcc(60, 60, 0.3, 2002)
    rA = D.rho_A(D.adjacency(g))
    ts = np.linspace(0.0, 10.0, 90)
    p, e, po, eo = _case(wl, g, [0.0], ("exp", 1.0 / rA), 0, 30, 8, ts, 2026)
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-8
    assert np.max(np.abs(e - eo)) < 1e-8 * np.max(np.abs(po)) + 1e-6 * np.max(eo)


# ---- the rational block Krylov variant (AAA poles + shifted MINRES solves; wl_xnystrace_exp_rational) ----

def _rational_case(wl, g, thetas, f, ti, M, ts, seed, poles=None, inner_tol=1e-14, **kw):
    A = D.adjacency(g)
    fo = {"exp": C.exp, "resolvent": C.resolvent}[f[0]](f[1])
    Lap = D.laplacian(A, 1.0 - thetas[ti], fo)
    Om = gg.vectors(g.n, M, seed)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=f, **kw)
    if poles is None:   # the library's AAA poles on [0, t* ρ] with its Gershgorin ρ bound (Alg. 1 line 3)
        poles = wl.aaa_exp_poles(max(ts) * op.laplacian_bound(ti))
    p, e, info = op.xnystrace_exp_rational(torch.from_numpy(Om).cuda(), ts, poles=poles, theta_index=ti,
                                           inner_tol=inner_tol, inner_maxit=2000)
    op.close()
    po, eo = T.xnystrace_exp_rational(Lap, Om, poles, ts)   # the same poles, dense solves
    return p, e, po, eo, info


def test_rational_karate_aaa_poles_vs_oracle(wl):
    """Fig. 4(a)-shape workload (karate, 𝕃 at θ = 1, t ∈ [0, 10]) with the first AAA poles (one real pole and
    one conjugate pair: a 10-dimensional space; all 13 would nearly exhaust n = 34 and make the reduced pencil
    Ĥ K̂⁻¹ ill-conditioned on both sides): the block rational Krylov estimate against the oracle's block
    rational Arnoldi with dense shifted solves."""
    g = gg.karate()
    rA = D.rho_A(D.adjacency(g))
    ts = np.linspace(0.0, 10.0, 30)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0], f=("exp", 1.0 / rA))
    poles = wl.aaa_exp_poles(max(ts) * op.laplacian_bound(0))[:2]
    op.close()
    assert poles[0].imag == 0 and poles[1].imag > 0
    p, e, po, eo, info = _rational_case(wl, g, [1.0, 0.0], ("exp", 1.0 / rA), 0, 2, ts, 11, poles=poles)
    assert info["inner_iters"] > 0
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-10
    assert np.max(np.abs(e - eo)) < 1e-10 * np.max(np.abs(po)) + 1e-8 * np.max(eo)


def test_rational_poles_real_pair_and_infinity(wl):
    """Every pole kind in one space: ∞, a real pole, a conjugate pair, on a multi-tile BA graph (NBT θ = 0)."""
    g = gg.barabasi_albert(1201, 3, 5)
    rA = D.rho_A(D.adjacency(g))
    ts = np.linspace(0.0, 4.0, 9)
    poles = np.array([np.inf, -2.5, -1.0 + 3.0j, 0.5 + 6.0j])
    p, e, po, eo, info = _rational_case(wl, g, [0.0], ("exp", 1.0 / rA), 0, 5, ts, 3, poles=poles)
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-10
    assert np.max(np.abs(e - eo)) < 1e-10 * np.max(np.abs(po)) + 1e-8 * np.max(eo)


@pytest.mark.slow
def test_rational_midsize_road_fig7_shape(wl):
    """The paper's §5.2 / Fig. 7 configuration shape — road-like grid, NBT, M = 30 probes, 90 t in [0, 100],
    AAA poles on [0, t* ρ] — on a graph the dense oracle handles (n ≈ 3.5e3)."""
    g = gg.grid_lcc(60, 60, 0.3, 2002)
    rA = D.rho_A(D.adjacency(g))
    ts = np.linspace(0.0, 100.0, 90)
    p, e, po, eo, info = _rational_case(wl, g, [0.0], ("exp", 1.0 / rA), 0, 30, ts, 2026)
    assert np.max(np.abs(p - po) / np.abs(po)) < 1e-10
    assert np.max(np.abs(e - eo)) < 1e-10 * np.max(np.abs(po)) + 1e-8 * np.max(eo)
