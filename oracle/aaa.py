"""AAA rational approximation and the poles of Alg. 1 line 3 — TEST INFRASTRUCTURE (oracle).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this module.  Plain fp64 NumPy / SciPy.

Alg. 1 (alg:trace_estimation), line 3: "Approximate the spectral radius ρ(𝔏) of 𝔏, and
build the poles {ξ_j} of rational approximation of exp(−x) on the interval [0, t* ρ(𝔏)]. Use AAA
[MR3805855]"; the text after it: "we select the poles using the AAA algorithm for rational
approximation.  The support points for the approximation are sampled from the interval [0, t* ρ(𝔏)]."

AAA (Nakatsukasa, Sète, Trefethen, SISC 2018 — the cited MR3805855), as its definition: the
barycentric approximant r(z) = N(z)/D(z), N(z) = Σ_j w_j f_j / (z − z_j), D(z) = Σ_j w_j / (z − z_j),
grown greedily — each step adds as support point the sample where |F − R| is largest, then takes w as
the right singular vector of the smallest singular value of the Loewner matrix
L_{ik} = (F_i − f_k)/(Z_i − z_k) over the non-support samples — until max|F − R| <= tol max|F|.
The poles are the zeros of D, i.e. the finite eigenvalues of the arrowhead pencil
(E, B) = ([[0, wᵀ], [1, diag(z)]], diag(0, 1, …, 1)).

Readings (R18):
* sample set: Z = {0} ∪ X·10^linspace(−10, 0, 2000) with X = t* ρ(𝔏) — the paper says only "sampled from
  the interval"; logarithmic spacing resolves the decay of exp(−x) near 0 on long intervals;
* tol = 1e-13 (relative); at most 30 support points;
* Froissart doublets (spurious pole–zero pairs of AAA, [MR3805855] §5) are poles whose residue
  |Res_ξ r| = |N(ξ)/D'(ξ)| is below 1e-13 max|F|; they are dropped, as are poles on the spectral
  interval [0, X] of the real axis (a shifted system 𝔏 − ξI would be singular there);
* a pole is real when |Im ξ| <= 1e-10 max(1, |ξ|); the others come in conjugate pairs (real f, real
  samples), each represented by its member with Im ξ > 0.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def aaa(Z, F, tol: float = 1e-13, mmax: int = 30):
    """AAA: support points z, values f, weights w, and the max error on the samples."""
    Z = np.asarray(Z, dtype=float)
    F = np.asarray(F, dtype=float)
    M = len(Z)
    J = np.ones(M, dtype=bool)               # samples that are not support points
    z, f = [], []
    C = np.zeros((M, 0))
    R = np.full(M, F.mean())
    w = np.zeros(0)
    err = np.inf
    for _ in range(mmax):
        j = int(np.argmax(np.abs(F - R)))
        z.append(Z[j])
        f.append(F[j])
        J[j] = False
        c = np.zeros(M)
        c[J] = 1.0 / (Z[J] - Z[j])           # Cauchy column (support rows are never used)
        C = np.column_stack([C, c])
        fa = np.asarray(f)
        L = F[J, None] * C[J] - C[J] * fa[None, :]           # Loewner matrix
        _, _, Vh = np.linalg.svd(L, full_matrices=False)
        w = Vh[-1]
        N = C @ (w * fa)
        D = C @ w
        R = F.copy()
        R[J] = N[J] / D[J]
        err = float(np.max(np.abs(F - R)))
        if err <= tol * np.max(np.abs(F)):
            break
    return np.asarray(z), np.asarray(f), w, err


def aaa_poles(z, f, w):
    """Poles of the barycentric approximant (finite eigenvalues of the arrowhead pencil) and residues."""
    m = len(z)
    E = np.zeros((m + 1, m + 1))
    E[0, 1:] = w
    E[1:, 0] = 1.0
    E[1:, 1:] = np.diag(z)
    B = np.eye(m + 1)
    B[0, 0] = 0.0
    ev = sla.eigvals(E, B)
    pol = ev[np.isfinite(ev)]
    d = pol[:, None] - z[None, :]
    N = (d ** -1) @ (w * f)
    Dp = -(d ** -2) @ w
    return pol, N / Dp


def exp_poles(xmax: float, tol: float = 1e-13):
    """The poles of Alg. 1 line 3 for the interval [0, xmax] (readings in the module docstring):
    one representative per conjugate pair (Im > 0) and the real poles, sorted by (|Im|, Re)."""
    Z = np.concatenate([[0.0], xmax * np.logspace(-10.0, 0.0, 2000)])
    F = np.exp(-Z)
    z, f, w, _ = aaa(Z, F, tol)
    pol, res = aaa_poles(z, f, w)
    keep = np.abs(res) >= 1e-13 * np.max(np.abs(F))
    real = np.abs(pol.imag) <= 1e-10 * np.maximum(1.0, np.abs(pol))
    on_interval = real & (pol.real >= 0.0) & (pol.real <= xmax)
    keep &= ~on_interval
    out = [complex(p.real, 0.0) if r else p for p, r in zip(pol[keep], real[keep]) if r or p.imag > 0]
    return np.array(sorted(out, key=lambda p: (abs(p.imag), p.real)), dtype=complex)
