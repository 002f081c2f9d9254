"""Walk counting (oracle tier 1 and 2).  TEST INFRASTRUCTURE — see oracle/__init__.py.

Paper passages:
* walks and A^k:   Def. def:walks_and_paths, Prop. pro:power-of-adjacency
* NBT counts p_k:  Def. def:NBT, p_0=I, p_1=A, p_2=A^2-D and eq:Br
* BTDW counts q_k: P:276-289 — every backtracking step (i_l = i_{l+2}) of a walk is
                   downweighted by 1-μ; q_0=I, q_1=A, q_2=A^2-μD and eq:qrec
                   q_{k+1} = A q_k + μ(μI - D) q_{k-1}.
Reading R2: eq:qrec is used for k >= 2 only (at k = 1 it would give
A^2 + μ^2 I - μD != q_2); the seeds q_0, q_1, q_2 are special-cased as the paper states.
"""
from __future__ import annotations

import numpy as np


def degree_matrix(A: np.ndarray) -> np.ndarray:
    """D with D_ii = (A 1)_i (Def. def:undirected_laplacian)."""
    return np.diag(A @ np.ones(A.shape[0]))


def brute_force_q(A: np.ndarray, mu: float, k: int) -> np.ndarray:
    """(q_k)_ij = Σ over all walks i=i_0,...,i_k=j of (1-μ)^{#{l : i_l = i_{l+2}}}.

    Exhaustive enumeration of walks (exponential cost; n <= 8, k <= 6).
    """
    n = A.shape[0]
    nbrs = [np.flatnonzero(A[i]) for i in range(n)]
    w = 1.0 - mu
    Q = np.zeros((n, n))

    def extend(walk, weight):
        if len(walk) == k + 1:
            Q[walk[0], walk[-1]] += weight
            return
        for j in nbrs[walk[-1]]:
            bt = len(walk) >= 2 and walk[-2] == j  # step i_l -> i_{l+1} -> i_{l+2} = i_l
            extend(walk + [int(j)], weight * (w if bt else 1.0))

    for i in range(n):
        extend([i], 1.0)
    return Q


def adjacency_powers(A: np.ndarray, K: int) -> list[np.ndarray]:
    """[A^0, ..., A^K] (Prop. pro:power-of-adjacency)."""
    out = [np.eye(A.shape[0])]
    for _ in range(K):
        out.append(A @ out[-1])
    return out


def nbt_p(A: np.ndarray, K: int) -> list[np.ndarray]:
    """[p_0, ..., p_K]: p_0=I, p_1=A, p_2=A^2-D, p_k = A p_{k-1} + (I-D) p_{k-2} for k >= 3 (eq:Br)."""
    n = A.shape[0]
    D = degree_matrix(A)
    I = np.eye(n)
    p = [I, A.copy(), A @ A - D]
    for k in range(3, K + 1):
        p.append(A @ p[k - 1] + (I - D) @ p[k - 2])
    return p[: K + 1]


def btdw_q(A: np.ndarray, mu: float, K: int) -> list[np.ndarray]:
    """[q_0, ..., q_K]: q_0=I, q_1=A, q_2=A^2-μD, q_{k+1} = A q_k + μ(μI - D) q_{k-1} for k >= 2 (eq:qrec)."""
    n = A.shape[0]
    D = degree_matrix(A)
    I = np.eye(n)
    q = [I, A.copy(), A @ A - mu * D]
    for k in range(2, K):
        q.append(A @ q[k] + mu * (mu * I - D) @ q[k - 1])
    return q[: K + 1]


def companion_Z(A: np.ndarray, mu: float) -> np.ndarray:
    """Z = [[O, I], [μ(μI - D), A]] (eq:Zdef), 2n x 2n."""
    n = A.shape[0]
    D = degree_matrix(A)
    I = np.eye(n)
    return np.block([[np.zeros((n, n)), I], [mu * (mu * I - D), A]])
