"""Pins for the CPU oracle: values the paper prints, brute force, closed forms, invariants.

Each test pins the oracle to something other than itself, chosen so that a plausible
mistake (dropped term, wrong sign/index, transposed operand, wrong seed) fails one of them.
"""
import math

import numpy as np
import pytest

import graphgen as gg
from oracle import coeffs as C
from oracle import dense as D
from oracle import walks as W
from conftest import read_golden

TS30 = np.linspace(0.0, 10.0, 30)


# ---------------------------------------------------------------- paper-printed values
def test_fig4a_karate_standard_laplacian_return_probability():
    """Fig. 4(a) 'True value': (1/n) tr exp(-tL), karate, n = 34 (reading R9)."""
    gold = np.array(read_golden("fig4a_karate_L_true.txt"), dtype=float)
    A = D.adjacency(gg.karate())
    # c = (0,1,0,...) gives 𝕃(c) = L: build it through the walk-Laplacian route
    Lap = D.walk_laplacian(D.phi_series(A, 0.0, C.monomial(1)))
    assert np.array_equal(Lap, D.standard_laplacian(A))
    ph = D.return_probability(Lap, gold[:, 0])
    assert np.allclose(gold[:, 0], TS30, atol=1e-13)
    assert np.max(np.abs(ph - gold[:, 1])) < 1e-13


def test_fig4b_karate_nbt_resolvent_return_probability():
    """Fig. 4(b) 'True value': 𝕃_1((1-αx)^-1), α = 1/(1+ρ(Z)) (caption P:1260).

    Reading R5: the printed curve uses the normalisation (1-α) instead of eq:katz-based-walk-
    laplacian's (1-α²), i.e. it is exp(-t 𝕃 /(1+α)); with (1-α²) the curve misses by ~0.04.
    """
    gold = np.array(read_golden("fig4b_karate_nbt_resolvent_true.txt"), dtype=float)
    A = D.adjacency(gg.karate())
    rz = D.rho_Z(A, 1.0)
    assert abs(rz - 5.292780644548677) < 1e-9
    alpha = 1.0 / (1.0 + rz)
    Lap = D.walk_laplacian(D.phi_resolvent_closed(A, 1.0, alpha))
    ph = D.return_probability(Lap / (1.0 + alpha), gold[:, 0])
    assert np.max(np.abs(ph - gold[:, 1])) < 5e-12
    ph_eq = D.return_probability(Lap, gold[:, 0])
    assert np.max(np.abs(ph_eq - gold[:, 1])) > 1e-2    # eq. (1-α²) does not reproduce the figure


def _fig1_panels():
    rows = read_golden("fig1_g58_stationary.txt")
    out = {}
    for name, node, val in rows:
        out.setdefault(name, np.zeros(13))[int(node) - 1] = float(val)
    return out


def test_fig1_trap_graph_stationary_distributions():
    """Fig. 1 on G_{5,8}: π ∝ t = f(A)1 for L, 𝕃(res) α=1/(2ρ(A)), 𝕃(exp) β=1.

    Reading R6: the printed bars equal t/Σt (D = diag(f(A)1)), not diag(𝕃)/Σ.
    """
    gold = _fig1_panels()
    A = D.adjacency(gg.trap_graph(5, 8))
    one = np.ones(13)
    rA = D.rho_A(A)
    assert abs(rA - 3.1964027540390294) < 1e-12
    t = {"L": A @ one,
         "res": D.phi(A, 0.0, C.resolvent(1.0 / (2.0 * rA))) @ one,
         "exp": D.phi(A, 0.0, C.exp(1.0)) @ one}
    for k, tv in t.items():
        assert np.max(np.abs(tv / tv.sum() - gold[k])) < 1e-14, k
    # exp panel also through the series route (independent of the eigendecomposition)
    ts = D.phi_series(A, 0.0, C.exp(1.0)) @ one
    assert np.max(np.abs(ts / ts.sum() - gold["exp"])) < 1e-14
    # the diag(𝕃) reading misses (documents reading R6)
    dL = np.diag(D.laplacian(A, 0.0, C.exp(1.0)))
    assert np.max(np.abs(dL / dL.sum() - gold["exp"])) > 1e-3


def test_fig1_trap_graph_nbt_exp_panel_bottom_block():
    """Fig. 1 𝕃_1(exp) panel: integers/674 = [O I] φ_1(Z)[d; A d - d], no c_0 term (reading R4).

    eq:exp-based-laplacian's top block [I O] gives a different vector; the figure was made
    with the bottom block, which equals Σ_{k>=2} p_k 1 / (k-1)!.  Pins Z, φ_1 and the seeds.
    """
    gold = _fig1_panels()["nbt_exp"]
    assert np.allclose(gold * 674, np.round(gold * 674), atol=1e-11)
    A = D.adjacency(gg.trap_graph(5, 8))
    one = np.ones(13)
    bot = D.phi_companion(A, 1.0, C.exp(1.0), block="bottom") @ one
    assert np.max(np.abs(bot / bot.sum() - gold)) < 1e-14
    # closed combinatorial form on the tree (p_k = 0 beyond the diameter 4)
    p = W.nbt_p(A, 8)
    assert np.all(p[5] == 0) and np.all(p[8] == 0)
    direct = sum(p[k] @ one / math.factorial(k - 1) for k in range(2, 6))
    assert np.max(np.abs(direct / direct.sum() - gold)) < 1e-14
    top = D.phi_companion(A, 1.0, C.exp(1.0), block="top") @ one
    assert np.max(np.abs(top / top.sum() - gold)) > 1e-2


# ---------------------------------------------------------------- brute force / recurrences
def _small_graphs():
    gs = [gg.path(3), gg.complete(3), gg.cycle(4), gg.star(4), gg.complete(4),
          gg.from_edges(10, [(i, (i + 1) % 5) for i in range(5)] + [(i, 5 + i) for i in range(5)]
                        + [(5 + i, 5 + (i + 2) % 5) for i in range(5)], "petersen")]
    rng = np.random.default_rng(11)
    for _ in range(8):
        n = 7
        e = [(i, j) for i in range(n) for j in range(i + 1, n) if rng.random() < 0.45]
        gs.append(gg.from_edges(n, e))
    return gs


@pytest.mark.parametrize("mu", [0.0, 0.25, 0.5, 0.75, 1.0])
def test_qrec_equals_brute_force_enumeration(mu):
    """eq:qrec with seeds q_0=I, q_1=A, q_2=A²-μD == weighted walk enumeration."""
    for g in _small_graphs():
        A = D.adjacency(g)
        kmax = 6 if g.n <= 7 else 4
        q = W.btdw_q(A, mu, kmax)
        for k in range(kmax + 1):
            bf = W.brute_force_q(A, mu, k)
            assert np.max(np.abs(q[k] - bf)) < 1e-12, (g.name, mu, k)


def test_recurrence_endpoints():
    """μ = 0 gives A^k (Prop. pro:power-of-adjacency); μ = 1 gives p_k of eq:Br."""
    for g in _small_graphs()[:8]:
        A = D.adjacency(g)
        q0, q1 = W.btdw_q(A, 0.0, 7), W.btdw_q(A, 1.0, 7)
        ak, pk = W.adjacency_powers(A, 7), W.nbt_p(A, 7)
        for k in range(8):
            assert np.array_equal(q0[k], ak[k]) and np.array_equal(q1[k], pk[k])


def test_spec_worked_examples():
    """Small hand-checkable values."""
    A = D.adjacency(gg.path(3))
    assert np.allclose(W.btdw_q(A, 0.5, 2)[2], [[0.5, 0, 1], [0, 1, 0], [1, 0, 0.5]], atol=0)
    K3 = D.adjacency(gg.complete(3))
    assert np.array_equal(W.nbt_p(K3, 3)[3], 2 * np.eye(3))
    assert abs(D.rho_A(D.adjacency(gg.star(9))) - 3.0) < 1e-12
    C4 = D.adjacency(gg.cycle(4))
    assert abs(D.rho_Z(C4, 1.0) - 1.0) < 1e-7
    for g in _small_graphs():
        A = D.adjacency(g)
        assert abs(D.rho_Z(A, 0.0) - D.rho_A(A)) < 1e-9   # Z block-triangular at μ = 0


def test_companion_powers_shift_the_sequence():
    """Z^k [q_1; q_2] = [q_{k+1}; q_{k+2}] (proof of Prop. pro:whe-we-converge)."""
    A = D.adjacency(gg.karate())
    for mu in (0.0, 0.3, 1.0):
        q = W.btdw_q(A, mu, 9)
        Z = W.companion_Z(A, mu)
        X = np.vstack([q[1], q[2]])
        for k in range(1, 7):
            X = Z @ X
            assert np.max(np.abs(X - np.vstack([q[k + 1], q[k + 2]]))) <= 1e-9 * np.max(np.abs(q[k + 2]))


# ---------------------------------------------------------------- closed forms / two routes
@pytest.mark.parametrize("mu", [0.0, 0.5, 1.0])
def test_phi_companion_route_equals_series(mu):
    """φ = [I O] f_1(Z)[q1;q2] + c0 I == Σ c_k q_k (series), exp β = 1/ρ(A)."""
    A = D.adjacency(gg.karate())
    f = C.exp(1.0 / D.rho_A(A))
    a, b = D.phi_companion(A, mu, f), D.phi_series(A, mu, f)
    assert np.max(np.abs(a - b)) < 1e-13 * np.max(np.abs(b))
    if mu == 0.0:
        c = D.phi_walk_eig(A, f)
        assert np.max(np.abs(c - b)) < 1e-13 * np.max(np.abs(b))


@pytest.mark.parametrize("mu", [0.0, 0.25, 0.5, 0.75, 1.0])
def test_resolvent_closed_form(mu):
    """(1-μ²α²)[(1-μ²α²)I - αA + μα²D]^{-1} == Σ α^k q_k == companion route; eq:deformed at μ=1."""
    A = D.adjacency(gg.karate())
    alpha = 0.5 / D.rho_A(A)
    f = C.resolvent(alpha)
    cf = D.phi_resolvent_closed(A, mu, alpha)
    assert np.max(np.abs(cf - D.phi_series(A, mu, f))) < 1e-13 * np.max(np.abs(cf))
    assert np.max(np.abs(cf - D.phi_companion(A, mu, f))) < 1e-12 * np.max(np.abs(cf))
    if mu == 1.0:
        lhs = cf @ D.deformed_laplacian(A, alpha)
        assert np.max(np.abs(lhs - (1 - alpha ** 2) * np.eye(34))) < 1e-13


def test_k3_resolvent_spec_example():
    """K3, μ=1, α=0.2: 𝒜 = 1.04 I - 0.2 A, φ = 0.96 𝒜^{-1}; eigenvalues 1.5, 0.96/1.24."""
    A = D.adjacency(gg.complete(3))
    ph = D.phi_resolvent_closed(A, 1.0, 0.2)
    ev = np.sort(np.linalg.eigvalsh(ph))
    assert np.allclose(ev, [0.96 / 1.24, 0.96 / 1.24, 1.5], atol=1e-14)


# ---------------------------------------------------------------- invariants of 𝕃
@pytest.mark.parametrize("mu", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("fkind", ["exp", "resolvent"])
def test_laplacian_invariants(mu, fkind):
    """Props. pro:still-an-mmatrix / pro:still-again-an-mmatrix."""
    for g in [gg.karate(), gg.trap_graph(5, 8), gg.grid(5, 6), gg.star(7)]:
        A = D.adjacency(g)
        rA = D.rho_A(A)
        f = C.exp(1.0 / rA) if fkind == "exp" else C.resolvent(0.5 / rA)
        ph = D.phi(A, mu, f)
        Lap = D.walk_laplacian(ph)
        t = ph @ np.ones(g.n)
        s = np.max(np.abs(Lap))
        assert np.max(np.abs(Lap @ np.ones(g.n))) < 1e-13 * s          # 𝕃 1 = 0
        assert np.max(np.abs(Lap - Lap.T)) < 1e-13 * s                  # symmetric
        off = Lap - np.diag(np.diag(Lap))
        assert np.max(off) <= 1e-15 * s                                 # M-matrix sign pattern
        ev = np.linalg.eigvalsh(Lap)
        assert ev[0] > -1e-12 * s and ev[-1] <= 2 * np.max(t - f.c(0)) * (1 + 1e-12)  # Gershgorin
        assert np.sum(ev < 1e-10 * s) == 1                              # connected: nullity 1


def test_reduction_to_standard_laplacian():
    """c = (0,1,0,...) ⇒ 𝕃(c) = L, for every μ (q_1 = A)."""
    A = D.adjacency(gg.karate())
    for mu in (0.0, 0.5, 1.0):
        assert np.array_equal(D.laplacian(A, mu, C.monomial(1)), D.standard_laplacian(A))


# ---------------------------------------------------------------- survey cross-check values
SURVEY_A11 = {  # karate, independent second implementation (60-term series)
    1.0: (75.8868438034475, 4.55866947675091, 8.41414239420315, 3.68050040868, 0.0743208776563225,
          58.4221805932838, 4.88684386709851),
    0.5: (74.0285144941793, 4.35678129883324, 8.20937951036889, 3.55690962077, 0.0778291231610663,
          56.5038878221236, 4.59009368017943),
    0.0: (72.2681395205439, 4.16543255340346, 8.02251122811095, 3.44200490262, 0.0814451742133106,
          54.8659591537328, 4.34571831275268),
}


@pytest.mark.parametrize("theta", [1.0, 0.5, 0.0])
def test_survey_karate_cross_check(theta):
    """θ = 1-μ.  Values from SURVEY App. A.11 (independent implementation)."""
    A = D.adjacency(gg.karate())
    rA = D.rho_A(A)
    mu = 1.0 - theta
    v = gg.vectors(34, 1, 101)[:, 0]
    assert v[0] == pytest.approx(-0.790152499963015, abs=1e-14)
    ph = D.phi(A, mu, C.exp(1.0 / rA))
    Lap = D.walk_laplacian(ph)
    t = ph @ np.ones(34)
    ref = SURVEY_A11[theta]
    assert t.sum() == pytest.approx(ref[0], rel=1e-12)
    assert t[0] == pytest.approx(ref[1], rel=1e-12)
    assert np.linalg.norm(Lap @ v) == pytest.approx(ref[2], rel=1e-12)
    assert np.linalg.eigvalsh(Lap)[-1] == pytest.approx(ref[3], rel=1e-10)
    x = D.diffusion(Lap, np.eye(34)[:, 0], [1.0])[:, 0]
    assert x[0] == pytest.approx(ref[4], rel=1e-12)
    phr = D.phi(A, mu, C.resolvent(0.5 / rA))
    assert (phr @ np.ones(34)).sum() == pytest.approx(ref[5], rel=1e-12)
    assert np.linalg.norm(D.walk_laplacian(phr) @ v) == pytest.approx(ref[6], rel=1e-12)


# ---------------------------------------------------------------- Markov chain (NEXT-3)
def test_fig1_markov_chain_stationary_by_eigenvector():
    """eq:let_there_be_markov: the chain P = I - D^{-1}𝕃 built by oracle/markov.py has the
    Fig. 1 bars as its stationary distribution, computed as a left eigenvector of P (independent of the
    t/Σt route of the test above).  Pins transition() and reading R6 (D = diag(t))."""
    from oracle import markov as M
    gold = _fig1_panels()
    A = D.adjacency(gg.trap_graph(5, 8))
    rA = D.rho_A(A)
    for key, f in (("res", C.resolvent(1.0 / (2.0 * rA))), ("exp", C.exp(1.0))):
        ph = D.phi(A, 0.0, f)
        t = ph @ np.ones(13)
        P = M.transition(D.walk_laplacian(ph), t)
        assert np.allclose(P.sum(1), 1.0, atol=1e-14) and P.min() >= -1e-15   # row-stochastic
        assert np.max(np.abs(M.stationary_eig(P) - gold[key])) < 1e-13, key
    # standard Laplacian panel: D = diag(L) = degrees, P = D^{-1}A (simple random walk)
    L = D.standard_laplacian(A)
    P = M.transition(L, A.sum(1))
    assert np.allclose(P, A / A.sum(1)[:, None])
    assert np.max(np.abs(M.stationary_eig(P) - gold["L"])) < 1e-13


def test_markov_evolution_invariants():
    """p_k keeps mass 1 and nonnegativity and converges to π ∝ t on a connected non-bipartite graph
    (karate) for every θ; one step equals the plain vector-matrix product."""
    from oracle import markov as M
    g = gg.karate()
    A = D.adjacency(g)
    for mu in (0.0, 0.5, 1.0):
        ph = D.phi(A, mu, C.exp(1.0 / D.rho_A(A)))
        t = ph @ np.ones(g.n)
        P = M.transition(D.walk_laplacian(ph), t)
        p0 = np.zeros(g.n)
        p0[0] = 1.0
        ps = M.evolve(P, p0, 200)
        assert np.allclose(ps.sum(1), 1.0, atol=1e-12) and ps.min() >= -1e-15
        assert np.allclose(ps[0], p0 @ (np.diag(1.0 / t) @ ph))
        assert np.max(np.abs(ps[-1] - t / t.sum())) < 1e-10
