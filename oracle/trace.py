"""Average return probability by Alg. 1 (XNysTrace-exp) — TEST INFRASTRUCTURE (oracle).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this module.  Plain fp64 NumPy / SciPy, in the order and notation of Alg. 1
(alg:trace_estimation) and the text after it:

1. Ω = [ω_1 … ω_M], iid isotropic probes.  The caller passes Ω in (Gaussian columns
   from ``graphgen.vectors``); E[ω ωᵀ] = I.
2. Block Krylov basis V_{k+1} and block Hessenberg pencil (𝓗_k, 𝒦_k) with 𝔏 V_{k+1} 𝒦_k =
   V_{k+1} 𝓗_k.  Reading R16: every pole ξ_j = ∞ — the
   definition allows "complex numbers or infinity" and then r_k ≡ 1, 𝒬^block_{k+1} is the
   polynomial block Krylov space span{Ω, 𝔏Ω, …, 𝔏^kΩ} (eq:block-rational-Krylov),
   𝒦_k = [I; 0] and the reduced pencil gives Ĥ_k 𝒦̂_k⁻¹ = H_k, the leading kM × kM block of 𝓗_k.
   The rational case, AAA poles (oracle/aaa.py) and shifted solves, is
   block_rational_arnoldi / xnystrace_exp_rational below.
3. Y(t) = (1/n) V_k exp(-t Ĥ_k 𝒦̂_k⁻¹) V_kᵀ Ω for every t.
4. p̂(t), ê(t) = XNysTrace(Y(t), Ω) ([XTRACE]).  Reading R17: the leave-one-out Nyström
   estimator of the cited work, written as its definition —
       Â_(i) = Y_{-i} (Ω_{-i}ᵀ Y_{-i})⁻¹ Y_{-i}ᵀ        (Nyström from the other M-1 probes)
       est_i = tr Â_(i) + ω_iᵀ (y_i − Â_(i) ω_i)       (exact part + Girard–Hutchinson residual)
       p̂ = mean_i est_i,   ê = std_i(est_i) / √M     (sample std, M-1 denominator)
   on the shifted matrix A_ν = A + νI, Y_ν = Y + νΩ, and p̂ ← p̂ − ν n (the stabilisation of the
   cited method).  ν = 1e-12 ‖Y‖_F / √M ≈ 1e-12 ‖A‖_F (E‖Aω‖² = ‖A‖_F²): large enough that
   Ω_{-i}ᵀ Y_ν,_{-i} stays numerically positive definite when A = exp(-t𝔏)/n is nearly rank one
   (its rounding is ~eps √M n ‖A‖_F against ν n), small enough to leave p̂ unchanged to ~1e-12.
   For M = 1 the Nyström part is empty (Â = 0) and est_1 = ω_1ᵀ y_1: Girard–Hutchinson.
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def xnystrace(Y: np.ndarray, Omega: np.ndarray) -> tuple[float, float]:
    """Trace estimate of the symmetric PSD A with Y = A Ω, and its error estimate (reading R17)."""
    n, M = Omega.shape
    nu = 1e-12 * np.linalg.norm(Y) / np.sqrt(M)
    Yn = Y + nu * Omega
    est = np.empty(M)
    for i in range(M):
        keep = [j for j in range(M) if j != i]
        Ym, Om = Yn[:, keep], Omega[:, keep]
        w, y = Omega[:, i], Yn[:, i]
        if keep:
            # Â_(i) = B Bᵀ with B = Y_{-i} C⁻ᵀ, C Cᵀ = Ω_{-i}ᵀ Y_{-i} (Cholesky): the same Nyström
            # approximation, in the form that stays accurate when A is (numerically) low rank.
            S = Om.T @ Ym
            C = np.linalg.cholesky(0.5 * (S + S.T))
            B = sla.solve_triangular(C, Ym.T, lower=True).T
            b = sla.solve_triangular(C, Ym.T @ w, lower=True)
            Ahat_tr = np.sum(B * B)                          # tr Â_(i)
            Ahat_ww = b @ b                                  # ω_iᵀ Â_(i) ω_i
        else:
            Ahat_tr, Ahat_ww = 0.0, 0.0
        est[i] = Ahat_tr + (w @ y - Ahat_ww)
    p = est.mean() - nu * n
    e = est.std(ddof=1) / np.sqrt(M) if M > 1 else 0.0
    return float(p), float(e)


def block_arnoldi(Lap: np.ndarray, Omega: np.ndarray, k: int):
    """Block Arnoldi with all poles at ∞ (reading R16): V_{k+1} (n × (k+1)M) orthonormal,
    𝓗_k ((k+1)M × kM) block upper Hessenberg with Lap V_k = V_{k+1} 𝓗_k, and R_0 with
    Ω = V_1 R_0.  Block Gram–Schmidt, applied twice (the orthogonalisation the paper leaves to
    [MR4082482]; it changes rounding only)."""
    n, M = Omega.shape
    V = np.zeros((n, (k + 1) * M))
    H = np.zeros(((k + 1) * M, k * M))
    Q, R0 = np.linalg.qr(Omega)
    V[:, :M] = Q
    for j in range(k):
        W = Lap @ V[:, j * M:(j + 1) * M]
        for _ in range(2):
            for i in range(j + 1):
                Vi = V[:, i * M:(i + 1) * M]
                C = Vi.T @ W
                H[i * M:(i + 1) * M, j * M:(j + 1) * M] += C
                W = W - Vi @ C
        Q, R = np.linalg.qr(W)
        V[:, (j + 1) * M:(j + 2) * M] = Q
        H[(j + 1) * M:(j + 2) * M, j * M:(j + 1) * M] = R
    return V, H, R0


def xnystrace_exp(Lap: np.ndarray, Omega: np.ndarray, k: int, ts) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 1 with poles at ∞: p̂(t), ê(t) for every t in ts.  Requires kM ≤ n (block Krylov space
    of full dimension; beyond n the basis breaks down)."""
    n, M = Omega.shape
    assert k * M <= n
    V, H, _ = block_arnoldi(Lap, Omega, k)
    Vk, Hk = V[:, :k * M], H[:k * M, :]
    p, e = np.empty(len(ts)), np.empty(len(ts))
    for s, t in enumerate(ts):
        Y = (1.0 / n) * (Vk @ (sla.expm(-t * Hk) @ (Vk.T @ Omega)))
        p[s], e[s] = xnystrace(Y, Omega)
    return p, e


def block_rational_arnoldi(Lap: np.ndarray, Omega: np.ndarray, poles):
    """Block rational Arnoldi ([MR4082482]) for the symmetric 𝔏 = Lap in REAL arithmetic.

    poles: sequence of ξ_j — np.inf, real numbers, or complex numbers standing for the conjugate pair
    {ξ, ξ̄} (real Ω, real 𝔏: the space with both poles has a real basis).  A final pole at ∞ is
    appended (reading R18: the reduced pencil Ĥ K̂⁻¹ is then the Rayleigh quotient V_kᵀ𝔏V_k).
    Step j takes the continuation block u = V c (the last M columns of the newest block — for a pair the
    imaginary part; the first M columns make the basis numerically unstable: a 1e-12 perturbation of the
    solves moved the smallest Ritz value by 30% on a 3.5e3-node road grid, reading R18) and
        ξ = ∞:      X = 𝔏 u                            𝔏 X-coefficients: K ← c,   H ← h
        ξ real:     X = (𝔏 − ξI)⁻¹ u   (dense solve)   𝔏 X = u + ξ X:  K ← h,   H ← c + ξ h
        ξ = a + ib: X = (𝔏 − ξI)⁻¹ u,  X ← [Re X, Im X]
                    𝔏 Xr = u + a Xr − b Xi, 𝔏 Xi = b Xr + a Xi:  K ← [hr hi], H ← [c + a hr − b hi, b hr + a hi]
    where X = V_new h after block classical Gram–Schmidt (applied twice) and a QR of the remainder, so
    𝔏 V K = V H holds column by column.  Returns V (n × D), K, H (D × (D − M)), R_0 (Ω = V_1 R_0)."""
    n, M = Omega.shape
    Q, R0 = np.linalg.qr(Omega)
    V = Q
    Kc, Hc = [], []                          # pencil columns (lengths grow with V)
    cstart = 0                               # continuation = columns [cstart, cstart + M) of V
    for xi in list(poles) + [np.inf]:
        if not np.iscomplex(xi):
            xi = float(np.real(xi))          # a real pole (possibly given with a zero imaginary part)
        D = V.shape[1]
        c = np.zeros((D, M))
        c[cstart:cstart + M] = np.eye(M)
        u = V @ c
        if np.isinf(xi):
            X = Lap @ u
        else:
            Xc = np.linalg.solve(Lap - xi * np.eye(n), u.astype(complex if np.iscomplex(xi) else float))
            X = np.hstack([Xc.real, Xc.imag]) if np.iscomplex(xi) else Xc
        m = X.shape[1]
        h = np.zeros((D + m, m))
        for _ in range(2):                   # block classical Gram–Schmidt, twice
            C = V.T @ X
            h[:D] += C
            X = X - V @ C
        Qn, Rn = np.linalg.qr(X)
        h[D:] = Rn
        V = np.hstack([V, Qn])
        cz = np.vstack([c, np.zeros((m, M))])
        if np.isinf(xi):
            Kc.append(cz)
            Hc.append(h)
        elif not np.iscomplex(xi):
            Kc.append(h)
            Hc.append(cz + xi * h)
        else:
            a, b = xi.real, xi.imag
            hr, hi = h[:, :M], h[:, M:]
            Kc.append(h)
            Hc.append(np.hstack([cz + a * hr - b * hi, b * hr + a * hi]))
        cstart = D + m - M                   # continuation: the LAST M columns of the newest block
    Dn = V.shape[1]
    K = np.hstack([np.vstack([k, np.zeros((Dn - k.shape[0], k.shape[1]))]) for k in Kc])
    H = np.hstack([np.vstack([x, np.zeros((Dn - x.shape[0], x.shape[1]))]) for x in Hc])
    return V, K, H, R0


def xnystrace_exp_rational(Lap: np.ndarray, Omega: np.ndarray, poles, ts) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 1 with the given poles: Y(t) = (1/n) V_k exp(−t Ĥ_k K̂_k⁻¹) V_kᵀ Ω, then
    XNysTrace (reading R17).  With the last pole at ∞ the reduced pencil Ĥ_k K̂_k⁻¹ IS the Rayleigh quotient
    V_kᵀ 𝔏 V_k (reading R18; the pin test_block_rational_arnoldi_decomposition_and_limits checks the
    identity on a well-conditioned case); it is evaluated in that form because K̂_k is ill-conditioned in
    floating point for spaces of many conjugate pairs."""
    n, M = Omega.shape
    V, K, H, _ = block_rational_arnoldi(Lap, Omega, poles)
    d = V.shape[1] - M
    Vk = V[:, :d]
    Ared = Vk.T @ Lap @ Vk
    p, e = np.empty(len(ts)), np.empty(len(ts))
    for s, t in enumerate(ts):
        Y = (1.0 / n) * (Vk @ (sla.expm(-t * Ared) @ (Vk.T @ Omega)))
        p[s], e[s] = xnystrace(Y, Omega)
    return p, e
