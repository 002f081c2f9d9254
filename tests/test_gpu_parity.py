"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Tolerance (BASELINE.json north_star): relative L2 error per column <= 1e-10 in fp64.
Sizes span several merge-path tiles and ragged tails; edge cases: isolated rows, zero
columns, breakdown (tiny / invariant Krylov spaces), chunking beyond 32 columns.
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


def _dense_case(wl, g, thetas, f, b, seed=101, **kw):
    A = D.adjacency(g)
    V = gg.vectors(g.n, b, seed)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=f, **kw)
    LV = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    PV = op.phi_apply(torch.from_numpy(V).cuda()).cpu().numpy()
    t = op.diag_shift().cpu().numpy()
    fo = {"exp": C.exp, "resolvent": C.resolvent}.get(f[0], C.series)(f[1])
    worst = 0.0
    for i, th in enumerate(thetas):
        ph = D.phi(A, 1.0 - th, fo)
        sl = slice(i * b, (i + 1) * b)
        worst = max(worst, relerr(LV[:, sl], D.walk_laplacian(ph) @ V).max(),
                    relerr(PV[:, sl], ph @ V).max(), relerr(t[:, i], ph.sum(1)).max())
    op.close()
    return worst


@pytest.mark.parametrize("b", [1, 8])
def test_karate_exp_three_variants(wl, b):
    """Config C1: walk (θ=1), θ=0.5 and nonbacktracking (θ=0), exp β = 1/ρ(A)."""
    g = gg.karate()
    beta = 1.0 / D.rho_A(D.adjacency(g))
    assert _dense_case(wl, g, [1.0, 0.5, 0.0], ("exp", beta), b) < TOL


def test_karate_variant_enums(wl):
    g = gg.karate()
    A = D.adjacency(g)
    beta = 1.0 / D.rho_A(A)
    V = gg.vectors(34, 2, 5)
    for variant, mu in (("walk", 0.0), ("nbt", 1.0)):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, variant=variant, f=("exp", beta))
        got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        assert relerr(got, D.laplacian(A, mu, C.exp(beta)) @ V).max() < TOL
        op.close()


def test_karate_resolvent_and_series(wl):
    g = gg.karate()
    rA = D.rho_A(D.adjacency(g))
    assert _dense_case(wl, g, [1.0, 0.25, 0.0], ("resolvent", 0.5 / rA), 3) < TOL
    assert _dense_case(wl, g, [0.7, 0.0], ("series", [0.5, 0.3, 0.2, 0.1, 0.05]), 2) < TOL


def test_reduction_to_standard_laplacian(wl):
    """c = (0, 1, 0, ...) gives 𝕃 = L = D - A for every θ."""
    g = gg.barabasi_albert(500, 3, 7)
    A = D.adjacency(g)
    V = gg.vectors(g.n, 4, 9)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0, 0.5, 0.0], f=("series", [0.0, 1.0]))
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    ref = D.standard_laplacian(A) @ V
    for i in range(3):
        assert relerr(got[:, 4 * i:4 * i + 4], ref).max() < 1e-13


def test_fig4b_through_gpu_operator(wl):
    """Materialise 𝕃_1((1-αx)^{-1}) on the GPU (34 unit vectors) and reproduce Fig. 4(b)."""
    from conftest import read_golden
    gold = np.array(read_golden("fig4b_karate_nbt_resolvent_true.txt"), dtype=float)
    g = gg.karate()
    A = D.adjacency(g)
    alpha = 1.0 / (1.0 + D.rho_Z(A, 1.0))
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, variant="nbt", f=("resolvent", alpha), krylov_dim=64)
    Lap = op.apply(torch.eye(34, dtype=torch.float64, device="cuda")).cpu().numpy()
    ph = D.return_probability(Lap / (1.0 + alpha), gold[:, 0])
    assert np.max(np.abs(ph - gold[:, 1])) < 1e-9
    t = op.diag_shift().cpu().numpy()
    op.close()
    # the same through the C ABI's 𝕃 scale (wl_walkfun.scale = 1/(1+α), reading R5), Krylov and CG solvers;
    # t = φ1 is not scaled
    for solver in ("krylov", "cg"):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, variant="nbt", f=("resolvent", alpha), krylov_dim=64,
                         lap_scale=1.0 / (1.0 + alpha), solver=solver, cg_tol=1e-14)
        Ls = op.apply(torch.eye(34, dtype=torch.float64, device="cuda")).cpu().numpy()
        assert np.max(np.abs(D.return_probability(Ls, gold[:, 0]) - gold[:, 1])) < 1e-9, solver
        assert np.allclose(op.diag_shift().cpu().numpy(), t, rtol=1e-10, atol=0)
        op.close()


@pytest.mark.parametrize("theta", [1.0, 0.5, 0.0])
def test_multi_tile_graphs_vs_series(wl, theta):
    """Power-law (R-MAT with isolated rows, hubs spanning tiles), BA and road-like graphs."""
    graphs = [gg.rmat(14, 12000, 150000, seed=21, perm_seed=22),
              gg.barabasi_albert(20000, 5, 31),
              gg.grid_lcc(150, 149, 0.3, 41)]
    for g in graphs:
        rA = S.rho_A(g)
        f = C.exp(1.0 / rA)
        for b in (1, 5):
            V = gg.vectors(g.n, b, 77)
            op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[theta], f=("exp", f.param))
            got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
            ref = S.laplacian_apply(g, 1.0 - theta, f, V, rA)
            assert relerr(got, ref).max() < TOL, (g.name, b)
            t = op.diag_shift().cpu().numpy()[:, 0]
            assert relerr(t, S.total_communicability(g, 1.0 - theta, f, rA)).max() < TOL
            op.close()


def test_theta_sweep_chunking_over_32_columns(wl):
    """11 θ values x b = 3 inputs = 33 output columns: two internal Krylov batches."""
    g = gg.rmat(12, 3000, 30000, seed=3, perm_seed=4)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    thetas = list(np.linspace(0.0, 1.0, 11))
    V = gg.vectors(g.n, 3, 8)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param))
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    for i, th in enumerate(thetas):
        ref = S.laplacian_apply(g, 1.0 - th, f, V, rA)
        assert relerr(got[:, 3 * i:3 * i + 3], ref).max() < TOL
    op.close()


def test_edge_cases(wl):
    # isolated rows and a zero column: φ v = c_0 v there, 𝕃 v = 0 on isolated rows
    g = gg.with_isolated(gg.karate(), 10)
    rA = S.rho_A(g)
    V = gg.vectors(g.n, 3, 1)
    V[:, 1] = 0.0
    V[:34, 2] = 0.0   # supported on isolated nodes only -> u = 0
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.5], f=("exp", 1.0 / rA))
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    ref = S.laplacian_apply(g, 0.5, C.exp(1.0 / rA), V, rA)
    assert relerr(got[:, [0]], ref[:, [0]]).max() < TOL
    assert np.all(got[:, 1] == 0.0) and np.all(got[:, 2] == 0.0)
    pv = op.phi_apply(torch.from_numpy(V).cuda()).cpu().numpy()
    assert np.array_equal(pv[:, 2], V[:, 2])
    op.close()
    # tiny graphs: Krylov space smaller than k (lucky breakdown), star with large k
    for g in (gg.path(2), gg.complete(3), gg.star(40)):
        rA = S.rho_A(g)
        for th in (1.0, 0.0):
            Vs = gg.vectors(g.n, 2, 3)
            op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[th], f=("exp", 1.0 / rA), krylov_dim=60)
            got = op.apply(torch.from_numpy(Vs).cuda()).cpu().numpy()
            ref = D.laplacian(D.adjacency(g), 1.0 - th, C.exp(1.0 / rA)) @ Vs
            assert relerr(got, ref).max() < TOL, (g.name, th)
            op.close()
    # edgeless graph: 𝕃 = 0
    e = gg.from_edges(5, [])
    op = wl.Operator(5, e.row_ptr, e.col_idx, thetas=[0.3], f=("exp", 1.0))
    assert np.all(op.apply(torch.ones(5, 1, dtype=torch.float64, device="cuda")).cpu().numpy() == 0)
    op.close()


def test_diffusion_karate_and_road(wl):
    """a9: exp(-τ𝕃)x0 vs dense eigendecomposition; Fig. 4 time grid."""
    for g, ts, kout in ((gg.karate(), np.linspace(0, 10, 30), 40),
                        (gg.grid_lcc(30, 30, 0.3, 5), np.linspace(0, 100, 19), 80)):
        A = D.adjacency(g)
        rA = D.rho_A(A)
        for th in (1.0, 0.0):
            x0 = np.zeros(g.n)
            x0[g.n // 2] = 1.0
            op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[th], f=("exp", 1.0 / rA))
            X = op.diffuse(torch.from_numpy(x0).cuda(), ts, k_out=kout).cpu().numpy()
            ref = D.diffusion(D.laplacian(A, 1.0 - th, C.exp(1.0 / rA)), x0, ts)
            assert relerr(X, ref).max() < TOL, (g.name, th)
            assert np.max(np.abs(X.sum(0) - 1.0)) < 1e-10        # mass conservation
            op.close()


def test_apply_host_matches_device(wl):
    g = gg.barabasi_albert(3000, 4, 2)
    rA = S.rho_A(g)
    V = gg.vectors(g.n, 2, 4)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0, 0.0], f=("exp", 1.0 / rA))
    a = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    b = op.apply_host(V)
    assert np.array_equal(a, b)   # same kernels, same order: bitwise
    op.close()


def test_cabi_errors(wl):
    g = gg.karate()
    with pytest.raises(wl.WalkLapError, match="WL_EINVAL"):
        wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.5], f=("exp", 1.0))
    bad = g.col_idx.copy()
    bad[0] = 0  # self loop on row 0
    with pytest.raises(wl.WalkLapError, match="WL_EGRAPH"):
        wl.Operator(g.n, g.row_ptr, bad, thetas=[1.0], f=("exp", 1.0))
    with pytest.raises(wl.WalkLapError, match="WL_EDIVERGE"):
        wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0], f=("resolvent", 0.2), rho_bound=6.73)


def test_full_c2_barabasi_albert(wl):
    """Config C2 at full size: BA n=1e5, avg degree 10, k=30, b=8, θ in {1, 0.5, 0}."""
    g = gg.barabasi_albert(100000, 5, 1001)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 8, 102)
    thetas = [1.0, 0.5, 0.0]
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param), krylov_dim=30)
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    for i, th in enumerate(thetas):
        ref = S.laplacian_apply(g, 1.0 - th, f, V, rA)
        assert relerr(got[:, 8 * i:8 * i + 8], ref).max() < TOL
    op.close()


def test_relabel_on_off_agree(wl):
    """Degree-sorted internal relabelling is invisible at the boundary (results in user order)."""
    g = gg.rmat(13, 6000, 60000, seed=5, perm_seed=6)
    rA = S.rho_A(g)
    V = gg.vectors(g.n, 3, 2)
    outs = []
    for rel in (0, 1):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.3, 1.0], f=("exp", 1.0 / rA), relabel=rel)
        outs.append((op.apply(torch.from_numpy(V).cuda()).cpu().numpy(), op.diag_shift().cpu().numpy()))
        x0 = np.zeros(g.n)
        x0[7] = 1.0
        outs[-1] += (op.diffuse(torch.from_numpy(x0).cuda(), [0.5, 2.0], k_out=30).cpu().numpy(),)
        op.close()
    for a, b in zip(outs[0], outs[1]):
        assert relerr(a, b).max() < 1e-12
    ref = S.laplacian_apply(g, 0.7, C.exp(1.0 / rA), V, rA)
    assert relerr(outs[1][0][:, :3], ref).max() < TOL


@pytest.mark.slow
def test_full_c4_theta_sweep_vs_series(wl):
    """Config C4 at full size (R-MAT n=1e7, nnz=4e8) in the bench launch configuration (11 θ, b=1,
    k=30): the θ ∈ {0, 0.5, 1} columns of the sweep vs the series oracle over all 1e7 rows, t_θ too.
    θ = 0 (nonbacktracking) is the numerically hardest column: |γ_i| = d_i - 1 reaches 3e5 against
    ρ(A) ≈ 3.4e3.  β = 1/ρ(A) with ρ(A) from the ORACLE (scipy Lanczos), passed to both sides (SURVEY
    §8(c) reading 8); the oracle's a-priori truncation bound uses ρ(A)(1 + 1e-3)."""
    from graphgen import configs
    cfg = configs.get("c4")
    g = cfg["make"]()
    A = S.csr(g)
    rho = S.rho_A(g, tol=1e-10)
    beta = 1.0 / rho
    V = gg.vectors(g.n, 1, cfg["vec_seed"])
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=cfg["thetas"], f=("exp", beta), krylov_dim=30)
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    t_gpu = op.diag_shift().cpu().numpy()
    op.close()
    # the adaptive-k bench line (bench.py --adaptive 1e-13): same workload, Arnoldi stopped by the estimate
    opa = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=cfg["thetas"], f=("exp", beta), krylov_dim=30,
                      krylov_tol=1e-13, krylov_adaptive=1)
    ws = opa.workspace(1)
    got_a = opa.apply(torch.from_numpy(V).cuda(), ws=ws).cpu().numpy()
    _, ksteps, kbatches = ws.stats()
    opa.close()
    assert ksteps / kbatches < 30
    f = C.exp(beta)
    ones_v = np.stack([np.ones(g.n), V[:, 0]], axis=1)
    for th in (0.0, 0.5, 1.0):
        i = cfg["thetas"].index(th)
        phi = S.phi_apply(g, 1.0 - th, f, ones_v, rho * 1.001, A=A)   # [t, φv] in one recurrence
        t = phi[:, 0]
        ref = t * V[:, 0] - phi[:, 1]
        assert relerr(t_gpu[:, i], t).max() < TOL, th
        assert relerr(got[:, i], ref).max() < TOL, th
        assert relerr(got_a[:, i], ref).max() < TOL, ("adaptive", th)
    # Σ_i (𝕃v)_i = tᵀv - 1ᵀφv = 0 for every θ column (φ symmetric, 1ᵀφ = tᵀ)
    for j in range(len(cfg["thetas"])):
        assert abs(got[:, j].sum()) < 1e-10 * np.abs(got[:, j]).sum()


@pytest.mark.slow
def test_full_c3_road_diffusion(wl):
    """Config C3 at full size (grid LCC n~2e6): NBT diffusion exp(-τ𝕃)x0 over the 90-point sweep
    τ in [0,100] (k_out = 80, the bench launch configuration); parity vs the Chebyshev oracle (SURVEY
    §8(c) tier 4) for every τ, and mass conservation 1ᵀx(τ) = 1ᵀx0."""
    from graphgen import configs
    from oracle import chebyshev
    g = configs.get("c3")["make"]()
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    taus = np.linspace(0.0, 100.0, 90)
    x0 = np.zeros(g.n)
    x0[g.n // 2] = 1.0
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, variant="nbt", f=("exp", f.param))
    X = op.diffuse(torch.from_numpy(x0).cuda(), taus, k_out=80).cpu().numpy()
    op.close()
    # the adaptive inner-k line (bench.py --diffusion --adaptive 1e-13)
    opa = wl.Operator(g.n, g.row_ptr, g.col_idx, variant="nbt", f=("exp", f.param), krylov_tol=1e-13,
                      krylov_adaptive=1)
    Xa = opa.diffuse(torch.from_numpy(x0).cuda(), taus, k_out=80).cpu().numpy()
    opa.close()
    assert np.max(np.abs(X.sum(axis=0) - 1.0)) < 1e-10          # mass 1ᵀx(τ) = 1ᵀx0
    ref = chebyshev.diffusion(g, 1.0, f, x0, taus, rA)
    assert relerr(X, ref).max() < TOL
    assert relerr(Xa, ref).max() < TOL


def test_apply_captured_in_cuda_graph(wl):
    """The whole 𝕃·V action is stream-ordered with no host synchronisation, so it captures into one CUDA graph
    (SURVEY §8(d) timing protocol); replays on new inputs match the oracle and the eager call bit for bit."""
    g = gg.rmat(14, 12000, 150000, seed=21, perm_seed=22)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    thetas = [0.0, 0.5, 1.0]
    b = 2
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param))
    ws = op.workspace(b)
    V = torch.from_numpy(gg.vectors(g.n, b, 5)).cuda()
    out = torch.empty((g.n, len(thetas) * b), dtype=torch.float64, device="cuda")
    op.apply(V, out=out, ws=ws)  # warm-up outside capture (one-time kernel attributes)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        op.apply(V, out=out, ws=ws)
    for seed in (6, 7):
        Vn = gg.vectors(g.n, b, seed)
        V.copy_(torch.from_numpy(Vn))
        graph.replay()
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        eager = op.apply(V, ws=ws).cpu().numpy()
        assert np.array_equal(got, eager)
        for i, th in enumerate(thetas):
            ref = S.laplacian_apply(g, 1.0 - th, f, Vn, rA)
            assert relerr(got[:, i * b:(i + 1) * b], ref).max() < TOL
    ws.close()
    op.close()


def test_spectral_radius_z_vs_dense(wl):
    """NEXT-4: ρ(Z_θ) by Arnoldi on the companion operator + host Hessenberg QR vs the dense eigenvalues
    of Z (oracle/dense.rho_Z); the karate NBT value is the one Fig. 4b's α uses (ρ(Z_1) = 5.29278...)."""
    g = gg.karate()
    A = D.adjacency(g)
    thetas = [0.0, 0.5, 1.0]
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", 0.1))
    for i, th in enumerate(thetas):
        got = op.spectral_radius_z(i, k=68)
        assert abs(got - D.rho_Z(A, 1.0 - th)) <= 1e-9 * got, th
    assert abs(op.spectral_radius_z(0, k=68) - 5.292780644548677) < 1e-9
    op.close()
    g = gg.barabasi_albert(400, 3, 11)
    A = D.adjacency(g)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", 0.1))
    for i, th in enumerate(thetas):
        got = op.spectral_radius_z(i, k=100)
        ref = D.rho_Z(A, 1.0 - th)
        assert abs(got - ref) <= 1e-8 * ref, (th, got, ref)
    op.close()


def test_markov_chain_vs_oracle(wl):
    """NEXT-3: p_{k+1} = p_k P, P = I - diag(t)^{-1}𝕃_θ (eq:let_there_be_markov, reading R6) vs the dense
    oracle chain (oracle/markov.py, pinned to Fig. 1); mass conservation; convergence to π = t/Σt."""
    from oracle import markov as M
    for g in (gg.karate(), gg.barabasi_albert(300, 3, 13)):
        A = D.adjacency(g)
        rA = D.rho_A(A)
        thetas = [0.0, 0.5, 1.0]
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", 1.0 / rA))
        p0 = gg.vectors(g.n, 1, 4)[:, 0] ** 2
        p0 /= p0.sum()
        for i, th in enumerate(thetas):
            ph = D.phi(A, 1.0 - th, C.exp(1.0 / rA))
            t = ph.sum(1)
            ref = M.evolve(M.transition(D.walk_laplacian(ph), t), p0, 6)
            got = op.markov(torch.from_numpy(p0).cuda(), 6, theta_index=i).cpu().numpy()
            assert relerr(got, ref.T).max() < TOL, (g.name, th)
            assert np.allclose(got.sum(0), 1.0, atol=1e-12)
        op.close()
    g = gg.karate()
    A = D.adjacency(g)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, variant="nbt", f=("resolvent", 0.5 / D.rho_A(A)))
    p0 = np.zeros(g.n)
    p0[0] = 1.0
    got = op.markov(torch.from_numpy(p0).cuda(), 300).cpu().numpy()
    t = op.diag_shift().cpu().numpy()[:, 0]
    assert np.max(np.abs(got[:, -1] - t / t.sum())) < 1e-9
    op.close()


@pytest.mark.parametrize("reorth", [1, 2])
@pytest.mark.parametrize("K", [1, 2, 7, 33, 64])
def test_orthogonalisation_variants_vs_series(wl, reorth, K):
    """Both basis schemes (opts.reorth: 1 = DCGS2 on 2n-vectors, 2 = TOAR on n-vectors) agree with the series
    oracle for small, odd, > 32 (tiled passes) and maximal Krylov dimensions; a ragged n*B forces the phantom row."""
    g = gg.barabasi_albert(3001, 4, 19)   # n odd
    rA = S.rho_A(g)
    f = C.exp(0.5 / rA)
    thetas = [0.0, 0.35, 1.0]
    b = 3                                   # B = 9 odd: n*B odd
    V = gg.vectors(g.n, b, 21)
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param), krylov_dim=K, reorth=reorth)
    got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
    worst = 0.0
    for i, th in enumerate(thetas):
        ref = S.laplacian_apply(g, 1.0 - th, f, V, rA)
        worst = max(worst, relerr(got[:, i * b:(i + 1) * b], ref).max())
    # k = 1, 2, 7 are genuine Krylov truncations (error ~1e-10 at k = 7): convergence, not parity
    tol = {1: 1e-1, 2: 1e-2, 7: 1e-8}.get(K, TOL)
    assert worst < tol, (reorth, K, worst)
    op.close()


def test_aposteriori_krylov_check(wl):
    """opts.tol (reading R11): a truncated Krylov space (k = 3) trips the sticky WL_ENOCONV reported by
    wl_wait, with the best iterate still written; a converged one (k = 30) does not, for both bases."""
    g = gg.karate()
    A = D.adjacency(g)
    beta = 1.0 / D.rho_A(A)
    V = torch.from_numpy(gg.vectors(g.n, 2, 3)).cuda()
    for reorth in (1, 2):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.5], f=("exp", beta), krylov_dim=3, krylov_tol=1e-12,
                         reorth=reorth)
        op.wait()  # operator creation (t) does not report
        got = op.apply(V).cpu().numpy()
        with pytest.raises(wl.WalkLapError) as e:
            op.wait()
        assert e.value.code == 4
        op.wait()  # cleared
        ref = D.laplacian(A, 0.5, C.exp(beta)) @ V.cpu().numpy()
        assert 1e-12 < relerr(got, ref).max() < 1e-1  # the truncated iterate is written
        op.close()
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.5], f=("exp", beta), krylov_dim=30, krylov_tol=1e-12,
                         reorth=reorth)
        op.apply(V)
        op.wait()
        op.close()


def test_hub_rows_split_into_chunks(wl):
    """Rows longer than the hub chunk (4096 nonzeros) are split across warps and reduced in chunk order by
    the last chunk to finish; several hubs of different lengths (1 to 3 chunks, and the boundary lengths) plus
    medium and small rows, vs the series."""
    rng = np.random.default_rng(5)
    n = 20000
    edges = set()
    for hub, deg in ((0, 10000), (1, 4097), (2, 8193), (3, 4096), (4, 700), (5, 2049), (6, 12289)):
        for v in rng.choice(np.arange(5, n), size=deg, replace=False):
            edges.add((min(hub, int(v)), max(hub, int(v))))
    for _ in range(20000):
        a, b = rng.integers(5, n, size=2)
        if a != b:
            edges.add((min(a, b), max(a, b)))
    g = gg.from_edges(n, sorted(edges), "hubs")
    assert np.diff(g.row_ptr).max() >= 12289
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 3, 8)
    for th in (0.0, 0.6):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[th], f=("exp", f.param))
        got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        assert relerr(got, S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() < TOL
        op.close()


@pytest.mark.parametrize("reorth", [1, 2])
def test_fuzz_small_graphs_exact_krylov(wl, reorth):
    """Randomised small cases (n <= 30, random density incl. isolated vertices, θ, walk function, b) with
    k = 64 >= 2n, where the Krylov space of Z is exhausted (lucky breakdown / U-level deflation paths): the
    action must equal the dense oracle to 1e-10 for both basis schemes."""
    rng = np.random.default_rng(1234 + reorth)
    for case in range(25):
        n = int(rng.integers(2, 31))
        p = float(rng.uniform(0.05, 0.6))
        e = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < p]
        if not e:
            e = [(0, 1)]
        g = gg.from_edges(n, e, f"fuzz{case}")
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
        thetas = list(np.round(rng.uniform(0, 1, size=int(rng.integers(1, 4))), 3))
        b = int(rng.integers(1, 4))
        V = gg.vectors(n, b, 100 + case)
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=f, krylov_dim=64, reorth=reorth)
        got = op.apply(torch.from_numpy(V).cuda()).cpu().numpy()
        for i, th in enumerate(thetas):
            ref = D.walk_laplacian(D.phi(A, 1.0 - th, fo)) @ V
            err = relerr(got[:, i * b:(i + 1) * b], ref).max()
            assert err < TOL, (case, n, kind, th, b, err)
        op.close()


@pytest.mark.slow
def test_full_c2_markov_vs_series(wl):
    """NEXT-3 at config C2 size (Barabási-Albert n = 1e5): three chain steps p_{k+1}^T = φ_θ (p_k / t) vs the series
    oracle (t and φ applies by the explicit recurrence); mass stays 1."""
    from graphgen import configs
    g = configs.get("c2")["make"]()
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    th = 0.5
    op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[th], f=("exp", f.param))
    p0 = gg.vectors(g.n, 1, 9)[:, 0] ** 2
    p0 /= p0.sum()
    got = op.markov(torch.from_numpy(p0).cuda(), 3).cpu().numpy()
    op.close()
    A = S.csr(g)
    t = S.total_communicability(g, 1.0 - th, f, rA, A=A)
    p = p0.copy()
    for k in range(3):
        p = S.phi_apply(g, 1.0 - th, f, p / t, rA, A=A)
        assert relerr(got[:, k], p).max() < TOL
        assert abs(got[:, k].sum() - 1.0) < 1e-12


def test_bitwise_reproducible_race_probe(wl):
    """compute-sanitizer is closed on this GPU pool (profiles/r02_compute_sanitizer_closed.log), so races are
    probed by determinism: every reduction on the path is fixed-order by design (per-CTA partials summed in CTA
    order, the hub-row chunks summed in chunk order by the last arriver, the mbarrier rings consumed in stage
    order), so repeated actions must agree BIT FOR BIT.  A hub with 9000 neighbours (three 4096-nonzero chunks and
    a ticket), 11 θ columns (32-byte lane gathers over the padded block), TOAR and DCGS2 rings, CG, diffusion."""
    r = gg.rmat(10, 900, 4000, seed=3, perm_seed=4)
    edges = [(int(i), int(j)) for i in range(r.n) for j in r.col_idx[r.row_ptr[i]:r.row_ptr[i + 1]] if i < j]
    n = r.n + 9001
    edges += [(r.n, r.n + 1 + k) for k in range(9000)] + [(0, r.n)]
    g = gg.from_edges(n, edges)
    rA = S.rho_A(g)
    V = torch.from_numpy(gg.vectors(n, 1, 5)).cuda()
    x0 = torch.zeros(n, dtype=torch.float64, device="cuda")
    x0[0] = 1.0
    for kw in (dict(reorth=2), dict(reorth=1), dict(solver="cg", f=("resolvent", 0.5 / rA))):
        kw.setdefault("f", ("exp", 1.0 / rA))
        op = wl.Operator(n, g.row_ptr, g.col_idx, thetas=[round(0.1 * i, 1) for i in range(11)], krylov_dim=16, **kw)
        outs = [op.apply(V).cpu().numpy() for _ in range(4)]
        if kw.get("solver") != "cg":
            outs += [op.diffuse(x0, [0.5, 2.0], k_out=12, theta_index=4).cpu().numpy() for _ in range(2)]
        op.close()
        for a, b in zip(outs[0:3], outs[1:4]):
            assert np.array_equal(a, b), kw
        if len(outs) > 4:
            assert np.array_equal(outs[4], outs[5]), kw


@pytest.mark.parametrize("f", [("exp", None), ("resolvent", None), ("series", [1.0, 0.5, 0.25, 0.125, 1.0 / 16])])
def test_lanczos_walk_path_vs_series(wl, f):
    """θ = 1 (all walks, μ = 0): batches whose columns are all θ = 1 take the symmetric Lanczos path
    (opts.lanczos); against the series oracle and against TOAR on Z (lanczos = 0), on power-law, BA
    and road-like graphs spanning many tiles, b = 3, plus t = φ1 at creation."""
    graphs = [gg.rmat(14, 12000, 150000, seed=21, perm_seed=22), gg.barabasi_albert(20000, 5, 31),
              gg.grid_lcc(150, 149, 0.3, 41)]
    for g in graphs:
        rA = S.rho_A(g)
        fo = C.exp(1.0 / rA) if f[0] == "exp" else C.resolvent(0.5 / rA) if f[0] == "resolvent" else C.series(f[1])
        fa = (f[0], fo.param if f[0] != "series" else f[1])
        V = gg.vectors(g.n, 3, 77)
        outs = []
        for lz in (1, 0):
            op = wl.Operator(g.n, g.row_ptr, g.col_idx, variant="walk", f=fa, lanczos=lz)
            outs.append((op.apply(torch.from_numpy(V).cuda()).cpu().numpy(), op.diag_shift().cpu().numpy()[:, 0]))
            op.close()
        ref = S.laplacian_apply(g, 0.0, fo, V, rA)
        assert relerr(outs[0][0], ref).max() < TOL, (g.name, f[0])
        assert relerr(outs[0][1], S.total_communicability(g, 0.0, fo, rA)).max() < TOL
        assert relerr(outs[0][0], outs[1][0]).max() < 1e-12


def test_adaptive_krylov_stop(wl):
    """opts.krylov_adaptive: the Arnoldi process stops at the first k' >= 6 where the a-posteriori estimate
    (reading R11) is below opts.tol for every column; the result still matches the series oracle (1e-10),
    and k' < krylov_dim on these graphs (k = 15 reaches 1.9e-16 on C2)."""
    graphs = [gg.rmat(14, 12000, 150000, seed=21, perm_seed=22), gg.grid_lcc(150, 149, 0.3, 41)]
    thetas = [0.0, 0.5, 0.8]
    for g in graphs:
        rA = S.rho_A(g)
        f = C.exp(1.0 / rA)
        V = gg.vectors(g.n, 2, 7)
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param), krylov_dim=40,
                         krylov_tol=1e-13, krylov_adaptive=1)
        ws = op.workspace(2)
        LV = op.apply(torch.from_numpy(V).cuda(), ws=ws).cpu().numpy()
        op.wait()
        _, steps, batches = ws.stats()
        op.close()
        assert steps / batches < 40, (g.name, steps, batches)
        for i, th in enumerate(thetas):
            assert relerr(LV[:, 2 * i:2 * i + 2], S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() < TOL, (g.name, th)


def test_isolated_tail_carries_no_krylov_data(wl):
    """wl_operator_active_rows: the relabelled isolated rows are left out of every Krylov vector (they vanish there,
    R13); φV = c_0 V and 𝕃V = 0 on them, the rest unchanged — against the oracle and against relabel = 0 (which
    keeps every row), for the TOAR and Lanczos batches and the fp32 mode."""
    g = gg.rmat(14, 12000, 150000, seed=21, perm_seed=22)
    deg = np.diff(g.row_ptr)
    rA = S.rho_A(g)
    f = C.exp(1.0 / rA)
    V = gg.vectors(g.n, 2, 5)
    thetas = [0.0, 0.5, 1.0]
    res = {}
    for rel in (1, 0):
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=thetas, f=("exp", f.param), relabel=rel)
        assert op.n_active == (int((deg > 0).sum()) if rel else g.n)
        res[rel] = (op.apply(torch.from_numpy(V).cuda()).cpu().numpy(), op.phi_apply(torch.from_numpy(V).cuda()).cpu().numpy())
        op.close()
    assert (deg == 0).sum() > 1000
    for a, b in zip(res[0], res[1]):
        assert relerr(a, b).max() < 1e-12
    LV, PV = res[1]
    iso = deg == 0
    assert np.all(LV[iso] == 0.0)
    assert np.array_equal(PV[iso], np.tile(V[iso], 3) * f.c(0))   # c_0 v exactly
    for i, th in enumerate(thetas):
        assert relerr(LV[:, 2 * i:2 * i + 2], S.laplacian_apply(g, 1.0 - th, f, V, rA)).max() < TOL, th
