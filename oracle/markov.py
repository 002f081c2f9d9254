"""Discrete-time Markov chain on a walk-based Laplacian (§3.x "Simulating discrete-time diffusion",
eq:let_there_be_markov) — TEST INFRASTRUCTURE (see oracle/__init__.py).

    P = I - D^{-1} 𝕃_μ(f),    p_{k+1} = p_k P,   p_0 1 = 1.

Reading R6: P:512 writes D = diag(𝕃_μ(f)), but P:515-516 says D "only requires a single
evaluation of the underlying matrix function", and Fig. 1's stationary bars equal t/Σt with
t = φ 1 (pinned in tests/test_oracle_pins.py).  Both point to D = diag(φ 1) = diag(t), which this
oracle takes.  Then P = diag(t)^{-1} φ is row-stochastic and π ∝ t is stationary (φ = φ^T).
"""
import numpy as np


def transition(lap: np.ndarray, t: np.ndarray) -> np.ndarray:
    """P = I - D^{-1} 𝕃 with D = diag(t) (eq:let_there_be_markov, reading R6); dense, small n."""
    n = lap.shape[0]
    return np.eye(n) - lap / t[:, None]


def evolve(P: np.ndarray, p0: np.ndarray, steps: int) -> np.ndarray:
    """Rows p_1 .. p_steps of p_{k+1} = p_k P (row vectors)."""
    out = []
    p = np.asarray(p0, dtype=float)
    for _ in range(steps):
        p = p @ P
        out.append(p)
    return np.array(out)


def stationary_eig(P: np.ndarray) -> np.ndarray:
    """π with π P = π, π 1 = 1, as the left eigenvector of P for the eigenvalue closest to 1
    (a route independent of t: used to pin π ∝ t against Fig. 1)."""
    w, V = np.linalg.eig(P.T)
    k = int(np.argmin(np.abs(w - 1.0)))
    v = np.real(V[:, k])
    return v / v.sum()
