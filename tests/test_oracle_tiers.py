"""Oracle tier consistency: the matrix-free series (tier 3) and the Chebyshev diffusion
(tier 4) — the routes used at the full configuration sizes — against the dense tier,
which is pinned to the paper in test_oracle_pins.py.  Also pins the input generators."""
import numpy as np
import pytest

import graphgen as gg
from oracle import chebyshev, coeffs as C, dense as D, series as S


def _graphs():
    return [gg.karate(),
            gg.barabasi_albert(300, 3, 5),
            gg.grid_lcc(18, 17, 0.3, 9),
            gg.with_isolated(gg.rmat(9, 400, 3000, seed=2, perm_seed=3), 7)]


@pytest.mark.parametrize("theta", [1.0, 0.5, 0.0])
def test_series_matches_dense(theta):
    mu = 1.0 - theta
    for g in _graphs():
        A = D.adjacency(g)
        rA = D.rho_A(A)
        assert abs(S.rho_A(g) - rA) < 1e-10 * rA
        V = gg.vectors(g.n, 3, 17)
        for f in (C.exp(1.0 / rA), C.resolvent(0.5 / rA), C.series([0.3, 0.2, 0.1, 0.05])):
            ph = D.phi(A, mu, f)
            ref = D.walk_laplacian(ph) @ V
            got = S.laplacian_apply(g, mu, f, V, rA)
            err = np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0)
            assert np.max(err) < 1e-13, (g.name, f.kind, err)
            t = S.total_communicability(g, mu, f, rA)
            assert np.max(np.abs(t - ph.sum(axis=1))) < 1e-13 * np.max(np.abs(t))


def test_series_isolated_rows_are_c0():
    """Isolated rows: q_k v vanishes there for k >= 1, so (φv)_i = c_0 v_i and (𝕃v)_i = 0."""
    g = gg.with_isolated(gg.karate(), 5)
    rA = S.rho_A(g)
    v = gg.vectors(g.n, 1, 3)[:, 0]
    f = C.exp(1.0 / rA)
    pv = S.phi_apply(g, 0.5, f, v, rA)
    assert np.array_equal(pv[34:], v[34:])
    assert np.all(S.laplacian_apply(g, 0.5, f, v, rA)[34:] == 0.0)


@pytest.mark.parametrize("theta", [1.0, 0.0])
def test_chebyshev_diffusion_matches_dense(theta):
    mu = 1.0 - theta
    g = gg.grid_lcc(20, 20, 0.3, 4)
    A = D.adjacency(g)
    rA = D.rho_A(A)
    f = C.exp(1.0 / rA)
    ts = np.linspace(0.0, 100.0, 19)
    x0 = np.zeros(g.n)
    x0[g.n // 2] = 1.0
    ref = D.diffusion(D.laplacian(A, mu, f), x0, ts)
    got = chebyshev.diffusion(g, mu, f, x0, ts, rA)
    err = np.linalg.norm(got - ref, axis=0) / np.linalg.norm(ref, axis=0)
    assert np.max(err) < 1e-12
    assert np.max(np.abs(got.sum(axis=0) - 1.0)) < 1e-12      # mass 1ᵀx(t) = 1ᵀx0
    # distance to the equilibrium (1ᵀx0 / n) 1 is nonincreasing in t (𝕃 symmetric PSD)
    dist = np.linalg.norm(ref - 1.0 / g.n, axis=0)
    assert np.all(np.diff(dist) <= 1e-14)


def test_generators_are_deterministic_and_simple():
    for make in (lambda: gg.rmat(12, 3000, 20000, seed=9, perm_seed=4),
                 lambda: gg.barabasi_albert(2000, 5, 1),
                 lambda: gg.grid_lcc(40, 41, 0.3, 2)):
        g1, g2 = make(), make()
        assert g1.sha256() == g2.sha256()
        rp, ci = g1.row_ptr, g1.col_idx
        rows = np.repeat(np.arange(g1.n), np.diff(rp))
        assert np.all(ci != rows)                                   # no loops
        key = rows.astype(np.int64) * g1.n + ci
        assert np.all(np.diff(key) > 0)                             # sorted, no duplicates
        keyT = ci.astype(np.int64) * g1.n + rows
        assert np.array_equal(np.sort(keyT), key)                   # symmetric
    g = gg.rmat(12, 3000, 20000, seed=9, perm_seed=4)
    assert g.nnz == 40000
    b = gg.barabasi_albert(2000, 5, 1)
    assert b.nnz == 2 * (5 + 5 * (2000 - 6))


def test_generator_thread_count_independence():
    import subprocess
    import sys
    code = ("import graphgen as gg; print(gg.rmat(14, 12000, 90000, seed=5, perm_seed=6).sha256(),"
            " gg.grid_lcc(60, 61, 0.3, 8).sha256())")
    outs = set()
    for t in ("1", "3"):
        env = dict(__import__("os").environ, OMP_NUM_THREADS=t)
        outs.add(subprocess.check_output([sys.executable, "-c", code], env=env,
                                         cwd=__import__("conftest").ROOT).strip())
    assert len(outs) == 1
