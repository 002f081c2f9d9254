"""Diffusion exp(-t𝕃) x0 at large n by a Chebyshev expansion (oracle tier 4).  TEST INFRASTRUCTURE.

Problem: p(t) = p_0 exp(-t 𝕃_μ(f)) (eq:diffusion_on_G_with_downweighted_walk);
𝕃 is symmetric so this is exp(-t𝕃) x0 with x0 = p_0^T.

Interval: Prop. pro:still-again-an-mmatrix gives σ(𝕃) ⊂ [0, 2 max(t - c_0)]
(Gershgorin with φ - c_0 I = Σ_{k>=1} c_k q_k >= 0).  With λ̄ = 2 max(t - c_0), s = 2x/λ̄ - 1
and τ = t λ̄ / 2 the Jacobi–Anger expansion gives

    exp(-t x) = ive(0, τ) T_0(s) + 2 Σ_{j>=1} (-1)^j ive(j, τ) T_j(s),

ive(j, τ) = I_j(τ) e^{-τ}.  The vectors T_j(Ŝ) x0, Ŝ = 2𝕃/λ̄ - I, do not depend on t, so every
t of the sweep accumulates in the same three-term Chebyshev recurrence.  ||T_j(Ŝ)||_2 <= 1,
so the truncation error is below Σ_{j>J} 2 ive(j, τ) ||x0||.
"""
from __future__ import annotations

import numpy as np
import scipy.special as ssp

from . import coeffs as C
from . import series


def diffusion(g, mu: float, f: C.WalkFun, x0: np.ndarray, ts, rho: float, tol: float = 1e-18,
              t_comm: np.ndarray | None = None) -> np.ndarray:
    """Columns exp(-t_s 𝕃) x0 for every t_s in ts."""
    A = series.csr(g)
    if t_comm is None:
        t_comm = series.total_communicability(g, mu, f, rho, A=A)
    tprime = t_comm - f.c(0)
    lam_bar = 2.0 * float(np.max(tprime)) if g.n > 0 else 1.0
    if lam_bar <= 0.0:
        return np.repeat(np.asarray(x0, float)[:, None], len(ts), axis=1)
    ts = np.asarray(ts, dtype=float)
    taus = ts * lam_bar / 2.0

    def Lapply(v):
        return t_comm * v - series.phi_apply(g, mu, f, v, rho, A=A)

    def S(v):                                  # Ŝ v = (2/λ̄) 𝕃 v - v
        return (2.0 / lam_bar) * Lapply(v) - v

    x0 = np.asarray(x0, dtype=float)
    out = np.zeros((g.n, len(ts)))
    T_prev, T_cur = x0, S(x0)
    out += ssp.ive(0, taus)[None, :] * T_prev[:, None]
    j = 1
    while True:
        cj = 2.0 * (-1.0) ** j * ssp.ive(j, taus)
        out += cj[None, :] * T_cur[:, None]
        # remaining tail is bounded by the next coefficients (decaying once j > τ)
        if j > np.max(taus) and np.max(np.abs(2.0 * ssp.ive(j + 1, taus))) * (j + 2) < tol:
            break
        T_prev, T_cur = T_cur, 2.0 * S(T_cur) - T_prev
        j += 1
        if j > 100000:
            raise RuntimeError("chebyshev: no convergence")
    return out
