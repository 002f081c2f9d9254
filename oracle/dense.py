"""Dense oracle (tier 2, n <= ~4096).  TEST INFRASTRUCTURE — see oracle/__init__.py.

Definitions followed:
* L = D - A                                          Def. def:undirected_laplacian
* φ_μ(A, c) = Σ_k c_k q_k(A)                         Prop. pro:whe-we-converge
* 𝕃_μ(c) = diag(φ 1) - φ                            eq:weighted_laplacian; μ=0 is
                                                     𝕃(f) = diag(f(A)1) - f(A) (eq:f-laplacian)
* φ = [I O] f_1(Z) [q_1; q_2] + c_0 I                Prop. pro:whe-we-converge
* resolvent, μ = 1: φ 𝒜(α) = (1-α^2) I              eq:deformed
* diffusion p(t) = p_0 exp(-t𝕃)                     P:131-141, eq:diffusion_on_G_with_downweighted_walk
* p̂_0(t) = (1/n) tr exp(-t𝔏)                        eq:average_return_probabilities
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import coeffs as C
from .walks import companion_Z, degree_matrix


def adjacency(g) -> np.ndarray:
    """Dense adjacency A_ij = 1 iff (i,j) in E (Def. def:adjacency) from a CSR pattern."""
    return g.dense()


def standard_laplacian(A: np.ndarray) -> np.ndarray:
    return degree_matrix(A) - A


def rho_A(A: np.ndarray) -> float:
    """Spectral radius of the symmetric adjacency (dense symmetric eigensolver)."""
    return float(np.max(np.abs(np.linalg.eigvalsh(A))))


def rho_Z(A: np.ndarray, mu: float) -> float:
    """ρ(Z) of the companion operator eq:Zdef (Table 1 reports it at μ = 1)."""
    return float(np.max(np.abs(np.linalg.eigvals(companion_Z(A, mu)))))


def phi_series(A: np.ndarray, mu: float, f: C.WalkFun, rho: float | None = None,
               tol: float = 1e-20) -> np.ndarray:
    """φ_μ(A,c) = Σ_{k=0}^{K} c_k q_k(A), q_k from eq:qrec, K from the a-priori tail bound.

    0 <= q_k <= A^k entrywise (weights (1-μ)^{#bt} in [0,1]) so ||q_k||_2 <= ρ(A)^k
    and Σ_{k>K} c_k ρ(A)^k bounds the truncation error.
    """
    n = A.shape[0]
    rho = rho_A(A) if rho is None else rho
    K = f.terms_needed(rho, tol)
    D = degree_matrix(A)
    I = np.eye(n)
    G = mu * (mu * I - D)
    q_prev, q = I, A.copy()                    # q_0, q_1
    phi = f.c(0) * q_prev + f.c(1) * q
    if K >= 2:
        q_prev, q = q, A @ A - mu * D          # q_2
        phi = phi + f.c(2) * q
    for k in range(2, K):
        q_prev, q = q, A @ q + G @ q_prev      # q_{k+1}
        phi = phi + f.c(k + 1) * q
    return phi


def phi_walk_eig(A: np.ndarray, f: C.WalkFun) -> np.ndarray:
    """μ = 0: φ = f(A) = V f(Λ) V^T (A symmetric; eq:f-laplacian)."""
    lam, V = np.linalg.eigh(A)
    return (V * C.scalar(f, lam)) @ V.T


def phi_resolvent_closed(A: np.ndarray, mu: float, alpha: float) -> np.ndarray:
    """Resolvent weights c_k = α^k for any μ (closed form derived from eq:qrec):

        ((1-μ²α²) I - α A + μ α² D) Φ = (1-μ²α²) I,   Φ = Σ_k α^k q_k.

    Derivation: sum eq:qrec times α^{k+1} over k >= 2 and use the seeds q_0, q_1, q_2.
    At μ = 1 this is eq:deformed with 𝒜(α) = I - αA - α²(I - D); at μ = 0 it is
    (I - αA)^{-1}.  Valid while α ρ(Z_μ) < 1 (Prop. pro:whe-we-converge).
    """
    n = A.shape[0]
    D = degree_matrix(A)
    s = 1.0 - mu * mu * alpha * alpha
    M = s * np.eye(n) - alpha * A + mu * alpha * alpha * D
    return s * np.linalg.inv(M)


def deformed_laplacian(A: np.ndarray, alpha: float) -> np.ndarray:
    """𝒜(α) = I - αA - α²(I - D)."""
    n = A.shape[0]
    return np.eye(n) - alpha * A - alpha ** 2 * (np.eye(n) - degree_matrix(A))


def phi_companion(A: np.ndarray, mu: float, f: C.WalkFun, block: str = "top") -> np.ndarray:
    """φ via the companion operator (Prop. pro:whe-we-converge):

        φ = [I O] f_1(Z) [q_1; q_2] + c_0 I,      f_1(x) = Σ_k c_{k+1} x^k  (eq:fs, s = 1).

    exp(βx): f_1(x) = β φ_1(βx), φ_1(x) = (e^x - 1)/x; φ_1(M) is the top-right
    block of expm([[M, I], [0, 0]]).  resolvent: f_1(x) = α (1 - αx)^{-1}.
    block="bottom" returns [O I] f_1(Z)[q_1; q_2] instead (reading R4: used only to reproduce
    the Fig. 1 NBT-exp panel, which the paper computed with the bottom block).
    """
    n = A.shape[0]
    D = degree_matrix(A)
    Z = companion_Z(A, mu)
    Q12 = np.vstack([A, A @ A - mu * D])           # [q_1; q_2]
    if f.kind == "exp":
        b = f.param
        aug = np.zeros((4 * n, 4 * n))
        aug[: 2 * n, : 2 * n] = b * Z
        aug[: 2 * n, 2 * n:] = np.eye(2 * n)
        F1 = b * sla.expm(aug)[: 2 * n, 2 * n:]   # β φ_1(βZ)
    elif f.kind == "resolvent":
        a = f.param
        F1 = a * np.linalg.inv(np.eye(2 * n) - a * Z)
    else:
        F1 = np.zeros((2 * n, 2 * n))
        Zm = np.eye(2 * n)
        for k in range(len(f.coeffs) - 1):
            F1 = F1 + f.c(k + 1) * Zm
            Zm = Zm @ Z
    if block == "top":
        return (F1 @ Q12)[:n] + f.c(0) * np.eye(n)
    return (F1 @ Q12)[n:]          # [O I] f_1(Z)[q_1; q_2] = Σ_{k>=0} c_{k+1} q_{k+2} (no c_0 I term)


def phi(A: np.ndarray, mu: float, f: C.WalkFun) -> np.ndarray:
    """Reference φ_μ(A, c) for small graphs: the exact definition, by the most direct route.

    resolvent -> closed form; μ = 0 exp/series -> eigen/series; otherwise the truncated series.
    """
    if f.kind == "resolvent":
        return phi_resolvent_closed(A, mu, f.param)
    if mu == 0.0 and f.kind == "exp":
        return phi_walk_eig(A, f)
    return phi_series(A, mu, f)


def walk_laplacian(phi_mat: np.ndarray) -> np.ndarray:
    """𝕃 = diag(φ 1) - φ (eq:f-laplacian / eq:weighted_laplacian)."""
    return np.diag(phi_mat @ np.ones(phi_mat.shape[0])) - phi_mat


def laplacian(A: np.ndarray, mu: float, f: C.WalkFun, scale: float = 1.0) -> np.ndarray:
    return scale * walk_laplacian(phi(A, mu, f))


def diffusion(Lap: np.ndarray, x0: np.ndarray, ts) -> np.ndarray:
    """exp(-t 𝕃) x0 for each t (columns), by the symmetric eigendecomposition of 𝕃.

    The paper's row-vector form p(t) = p_0 exp(-t𝕃) equals (exp(-t𝕃) p_0^T)^T since 𝕃 = 𝕃^T.
    """
    Ls = 0.5 * (Lap + Lap.T)
    lam, V = np.linalg.eigh(Ls)
    c = V.T @ x0
    return np.stack([V @ (np.exp(-t * lam) * c) for t in ts], axis=1)


def return_probability(Lap: np.ndarray, ts) -> np.ndarray:
    """p̂_0(t) = (1/n) Σ_i exp(-t λ_i) (eq:average_return_probabilities; exact)."""
    lam = np.linalg.eigvalsh(0.5 * (Lap + Lap.T))
    return np.array([np.mean(np.exp(-t * lam)) for t in ts])
