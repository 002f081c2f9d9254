"""Pins for oracle/trace.py (Alg. 1, XNysTrace-exp; readings R16/R17 in DESIGN.md §3).

Each pin fixes the oracle against something other than itself:
* low-rank exactness of the Nyström estimator (rank(A) < M-1 ⇒ Â_(i) = A, every est_i = tr A);
* M = 1 reduces to the textbook Girard–Hutchinson estimator ωᵀAω;
* unbiasedness over many seeded draws (a dropped residual term ω_iᵀ(A − Â_(i))ω_i biases low);
* the block Arnoldi relation and orthonormality, and exactness of Y(t) once kM ≥ n;
* the printed Fig. 4(a) 'True value' curve (tests/golden) within the estimator's own
  error estimate.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import graphgen as gg
from oracle import coeffs as C
from oracle import dense as D
from oracle import trace as T
from conftest import read_golden


def _psd(n, rank, seed):
    G = np.random.default_rng(seed).standard_normal((n, rank))
    return G @ G.T


def test_xnystrace_exact_for_low_rank():
    for n, r, M in [(40, 2, 5), (30, 1, 3), (25, 4, 6)]:
        A = _psd(n, r, 11 + r)
        Om = gg.vectors(n, M, 5 + M)
        p, e = T.xnystrace(A @ Om, Om)
        # exact up to the stabilising shift: cond(Ω_{-i}ᵀY_ν) ~ ‖A‖/ν = 1e12 costs ~1e-7 relative
        assert abs(p - np.trace(A)) <= 1e-6 * np.trace(A), (n, r, M)
        assert e <= 1e-6 * np.trace(A)


def test_xnystrace_single_probe_is_girard_hutchinson():
    A = _psd(30, 30, 3)
    om = gg.vectors(30, 1, 9)
    p, e = T.xnystrace(A @ om, om)
    assert abs(p - float(om[:, 0] @ A @ om[:, 0])) <= 1e-10 * abs(p)   # ν(‖ω‖² − n) ~ 1e-11
    assert e == 0.0


def test_xnystrace_unbiased_over_seeds():
    n, M, draws = 24, 4, 3000
    lam = np.exp(-np.linspace(0, 4, n))             # decaying PSD spectrum, like exp(-tL)
    Q = np.linalg.qr(np.random.default_rng(1).standard_normal((n, n)))[0]
    A = (Q * lam) @ Q.T
    est = np.array([T.xnystrace(A @ gg.vectors(n, M, s), gg.vectors(n, M, s))[0] for s in range(draws)])
    assert abs(est.mean() - lam.sum()) <= 4.0 * est.std(ddof=1) / np.sqrt(draws)
    # the Nyström part alone (residual term dropped) is biased low by far more than that
    hut = np.array([np.trace(A @ gg.vectors(n, M, s) @ np.linalg.solve(
        gg.vectors(n, M, s).T @ A @ gg.vectors(n, M, s), gg.vectors(n, M, s).T @ A))
        for s in range(200)])
    assert lam.sum() - hut.mean() > 0.05 * lam.sum()


def test_block_arnoldi_relation():
    A = D.adjacency(gg.karate())
    L = D.standard_laplacian(A)
    Om = gg.vectors(34, 3, 4)
    V, H, R0 = T.block_arnoldi(L, Om, 5)
    assert np.allclose(V.T @ V, np.eye(V.shape[1]), atol=1e-12)
    assert np.allclose(L @ V[:, :15], V @ H, atol=1e-11)
    assert np.allclose(V[:, :3] @ R0, Om, atol=1e-12)
    # symmetric 𝔏 ⇒ block tridiagonal H
    assert np.max(np.abs(H[:15][np.triu_indices(15, 4)])) < 1e-11


def test_y_exact_when_block_space_is_full():
    A = D.adjacency(gg.karate())
    L = D.standard_laplacian(A)
    Om = gg.vectors(34, 17, 21)
    V, H, _ = T.block_arnoldi(L, Om, 2)                # 2·17 = 34 = n: the whole space
    k, M, n = 2, 17, 34
    for t in (0.0, 0.5, 3.0):
        Y = V[:, :k * M] @ sla.expm(-t * H[:k * M]) @ V[:, :k * M].T @ Om / n
        assert np.allclose(Y, sla.expm(-t * L) @ Om / n, atol=1e-12)


def test_fig4a_within_error_estimate():
    """Fig. 4(a): karate, standard L, 30 t-points on [0,10] (caption P:1463).

    M = 17 probes, k = 2 blocks: kM = 34 = n, so Y(t) is exact and only the estimator is random.
    Over 10 seeded draws: the estimate lies within 3ê of the printed curve at ≥ 90% of the grid
    for ≥ 8 draws, and the mean over draws is within 0.03 everywhere."""
    gold = np.array(read_golden("fig4a_karate_L_true.txt"), dtype=float)
    L = D.standard_laplacian(D.adjacency(gg.karate()))
    ps, good = [], 0
    for seed in range(10):
        p, e = T.xnystrace_exp(L, gg.vectors(34, 17, seed), 2, gold[:, 0])
        ps.append(p)
        good += np.mean(np.abs(p - gold[:, 1]) <= 3 * e + 1e-12) >= 0.9
    assert good >= 8
    assert np.max(np.abs(np.mean(ps, axis=0) - gold[:, 1])) < 0.03


# ---- rational part of Alg. 1: AAA poles (oracle/aaa.py) and the block rational Arnoldi (oracle/trace.py) ----

def _lsq_rational_error(poles, X):
    """Max error on the AAA sample set of the least-squares fit of exp(-x) by 1 + Σ_j c_j/(x − ξ_j) over the
    poles and their conjugates: small iff the poles carry a rational approximation of exp(-x) on [0, X]."""
    from oracle import aaa as AA  # noqa: F401
    Z = np.concatenate([[0.0], X * np.logspace(-10.0, 0.0, 2000)])
    allp = []
    for p in poles:
        allp.append(p)
        if p.imag != 0:
            allp.append(np.conj(p))
    B = np.column_stack([np.ones_like(Z)] + [1.0 / (Z - p) for p in allp]).astype(complex)
    c, *_ = np.linalg.lstsq(B, np.exp(-Z).astype(complex), rcond=None)
    return float(np.abs(B @ c - np.exp(-Z)).max())


def test_aaa_recovers_the_poles_of_a_rational_function():
    """AAA is exact on a rational function (its closed form): 1/(x+2) + 3/(x+5) − 1/(x−12) sampled on [0, 10]."""
    from oracle import aaa as AA
    Z = np.linspace(0.0, 10.0, 500)
    F = 1.0 / (Z + 2.0) + 3.0 / (Z + 5.0) - 1.0 / (Z - 12.0)
    z, f, w, err = AA.aaa(Z, F)
    pol, res = AA.aaa_poles(z, f, w)
    assert err < 1e-13
    order = np.argsort(pol.real)
    assert np.allclose(pol[order].real, [-5.0, -2.0, 12.0], atol=1e-9) and np.all(np.abs(pol.imag) < 1e-9)
    assert np.allclose(res[order].real, [3.0, 1.0, -1.0], atol=1e-8)


@pytest.mark.parametrize("X", [10.0, 100.0, 1000.0])
def test_aaa_exp_poles_carry_the_approximation(X):
    """The poles of Alg. 1 line 3 support a rational approximation of exp(-x) on [0, X] to ~1e-13, come as
    conjugate pairs / real poles off the spectral interval; t* = 100 gives 13 poles counting conjugates,
    the count the paper reports for its road networks."""
    from oracle import aaa as AA
    poles = AA.exp_poles(X)
    assert _lsq_rational_error(poles, X) < 1e-12
    assert np.all(poles.imag >= 0)
    assert not np.any((poles.imag == 0) & (poles.real >= 0) & (poles.real <= X))
    if X == 100.0:
        assert sum(2 if p.imag > 0 else 1 for p in poles) == 13


def test_block_rational_arnoldi_decomposition_and_limits():
    """𝔏 V K = V H with V orthonormal for ∞ / real / complex-pair poles; all poles at ∞ reproduce the polynomial
    block Arnoldi estimate; the space is exact for f(x) = 1/(x − ξ) at each of its poles (rational Krylov
    exactness)."""
    g = gg.karate()
    A = D.adjacency(g)
    Lap = D.laplacian(A, 1.0, C.exp(1.0 / D.rho_A(A)))
    Om = gg.vectors(34, 3, 5)
    V, K, H, _ = T.block_rational_arnoldi(Lap, Om, [-2.0, 1.5 + 3.0j, np.inf])
    assert np.abs(Lap @ V @ K - V @ H).max() < 1e-13
    assert np.abs(V.T @ V - np.eye(V.shape[1])).max() < 1e-13
    d = V.shape[1] - 3                     # last pole ∞: reduced pencil = Rayleigh quotient (reading R18)
    assert np.abs(H[:d] @ np.linalg.inv(K[:d]) - V[:, :d].T @ Lap @ V[:, :d]).max() < 1e-12
    ts = np.linspace(0.0, 10.0, 5)
    p1, e1 = T.xnystrace_exp(Lap, Om, 3, ts)
    p2, e2 = T.xnystrace_exp_rational(Lap, Om, [np.inf, np.inf], ts)
    assert np.abs(p1 - p2).max() < 1e-13 and np.abs(e1 - e2).max() < 1e-13
    for xi in (-2.0, 0.7 + 2.0j):
        V, K, H, _ = T.block_rational_arnoldi(Lap, Om, [-2.0, 0.7 + 2.0j])
        d = V.shape[1] - 3
        Vk = V[:, :d]
        Ar = H[:d] @ np.linalg.inv(K[:d])
        for x in (xi, np.conj(xi)):
            approx = Vk @ np.linalg.solve(Ar - x * np.eye(d), Vk.T @ Om)
            exact = np.linalg.solve(Lap - x * np.eye(34), Om)
            assert np.abs(approx - exact).max() < 1e-12 * np.abs(exact).max()
