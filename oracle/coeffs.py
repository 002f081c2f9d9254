"""Walk weights {c_k} (Def. def:transformedlaplacian).  TEST INFRASTRUCTURE.

* exp with inverse temperature β: f(x) = exp(βx), c_k = β^k / k!  (remedy P:543)
* resolvent: c = (1, α, α^2, ...), f(x) = (1 - αx)^{-1}
* explicit series c_0..c_K (zero beyond K)                         (Def. def:transformedlaplacian)
* monomial e_j: c = (0,..,1,..0); c = (0,1,0,...) gives 𝕃(c) = L
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class WalkFun:
    kind: str                    # "exp" | "resolvent" | "series"
    param: float = 1.0           # β for exp, α for resolvent
    coeffs: tuple = field(default_factory=tuple)  # c_0..c_K for "series"

    def c(self, k: int) -> float:
        if self.kind == "exp":
            return self.param ** k / math.factorial(k) if k < 171 else 0.0
        if self.kind == "resolvent":
            return self.param ** k
        if self.kind == "series":
            return float(self.coeffs[k]) if k < len(self.coeffs) else 0.0
        raise ValueError(self.kind)

    def terms_needed(self, rho: float, tol: float = 1e-20) -> int:
        """Smallest K with Σ_{k>K} c_k ρ^k <= tol (a-priori tail bound; ρ >= ρ(A) bounds q_k)."""
        if self.kind == "series":
            return len(self.coeffs) - 1
        if self.kind == "resolvent":
            r = self.param * rho
            if r >= 1.0:
                raise ValueError("resolvent series bound needs α ρ(A) < 1 (use the closed form)")
            # tail = r^{K+1} / (1 - r)
            return max(2, int(math.ceil(math.log(tol * (1 - r)) / math.log(r))))
        if self.kind == "exp":
            x = self.param * rho
            K = 2
            # tail <= term_{K+1} / (1 - x/(K+2)) once K+2 > x
            while True:
                term = math.exp((K + 1) * math.log(max(x, 1e-300)) - math.lgamma(K + 2)) if x > 0 else 0.0
                if K + 2 > 2 * x and term <= tol * (1 - x / (K + 2)):
                    return K
                K += 1
        raise ValueError(self.kind)


def exp(beta: float) -> WalkFun:
    return WalkFun("exp", float(beta))


def resolvent(alpha: float) -> WalkFun:
    return WalkFun("resolvent", float(alpha))


def series(cs) -> WalkFun:
    return WalkFun("series", 0.0, tuple(float(x) for x in cs))


def monomial(j: int) -> WalkFun:
    return series([0.0] * j + [1.0])


def scalar(f: WalkFun, x) -> np.ndarray:
    """f(x) = Σ c_k x^k evaluated in closed form (used for eigenvalue-based dense evaluation, μ = 0)."""
    x = np.asarray(x, dtype=float)
    if f.kind == "exp":
        return np.exp(f.param * x)
    if f.kind == "resolvent":
        return 1.0 / (1.0 - f.param * x)
    return sum(c * x ** k for k, c in enumerate(f.coeffs))
