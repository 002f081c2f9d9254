"""Workload recipes of BASELINE.json configs C1..C5; inputs only.

Each entry builds the graph with the shared seeded generators and states the run parameters.
The *_mini variants keep the generator, degree structure and parameters at a size the CPU oracle
handles in seconds (used by tests).
"""
from __future__ import annotations

from . import barabasi_albert, grid_lcc, karate, rmat

THETA_SWEEP = [round(0.1 * i, 1) for i in range(11)]   # θ in {0, 0.1, ..., 1} (Fig. 6 palette)

CONFIGS = {
    "c1": dict(desc="Zachary karate club (n=34, m=78)", make=lambda: karate(),
               thetas=[1.0, 0.5, 0.0], b=8, krylov_dim=30, vec_seed=101),
    "c2": dict(desc="Barabasi-Albert n=1e5, m0=5 (avg degree 10), seed 1001",
               make=lambda: barabasi_albert(100000, 5, 1001),
               thetas=[1.0, 0.5, 0.0], b=8, krylov_dim=30, vec_seed=102),
    "c3": dict(desc="2D grid 1415x1414, 30% edge deletion, largest component, seed 2002",
               make=lambda: grid_lcc(1415, 1414, 0.3, 2002),
               thetas=[0.0], b=1, krylov_dim=30, vec_seed=None, k_out=80,
               taus=("linspace", 0.0, 100.0, 90)),
    "c4": dict(desc="R-MAT (0.57,0.19,0.19,0.05) scale 24 -> n=1e7, m=2e8 (nnz 4e8), seed 3003, "
                    "permuted ids (seed 7)",
               make=lambda: rmat(24, 10_000_000, 200_000_000, seed=3003, perm_seed=7),
               thetas=THETA_SWEEP, b=1, krylov_dim=30, vec_seed=103),
    "c5": dict(desc="R-MAT scale 26 -> n=5e7, m=1e9 (nnz 2e9), seed 4004, permuted ids",
               make=lambda: rmat(26, 50_000_000, 1_000_000_000, seed=4004, perm_seed=7),
               thetas=[0.5], b=32, krylov_dim=30, vec_seed=104),
    # reduced-size stand-ins with the same generators (tests, quick benches)
    "c4_mini": dict(desc="R-MAT scale 20 -> n=1e6, m=2e7, seed 3003, permuted ids",
                    make=lambda: rmat(20, 1_000_000, 20_000_000, seed=3003, perm_seed=7),
                    thetas=THETA_SWEEP, b=1, krylov_dim=30, vec_seed=103),
    "c3_mini": dict(desc="2D grid 300x300, 30% deletion, LCC, seed 2002",
                    make=lambda: grid_lcc(300, 300, 0.3, 2002),
                    thetas=[0.0], b=1, krylov_dim=30, vec_seed=None, k_out=80,
                    taus=("linspace", 0.0, 100.0, 90)),
}


def get(name: str) -> dict:
    return CONFIGS[name]
