"""CPU oracle for the walk-based Laplacians of arXiv 2601.11338 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import, call or execute anything in this package.
The product path (``paper_2601_11338_b200``) never imports it and shares no
code, header, table or helper with it; the only shared code is the seeded input
generator package ``graphgen`` (graphs + vectors, no method arithmetic).

Everything is plain fp64 NumPy / SciPy, written to be checked against the
paper by eye:

* ``walks``     — walk counts: brute-force enumeration, A^k
                  (Prop. pro:power-of-adjacency), NBT p_k (eq:Br,
                  P:269-272) and BTDW q_k (eq:qrec).
* ``coeffs``    — the walk weights c_k of the functions used in the paper
                  (exp with inverse temperature, resolvent, explicit series).
* ``dense``     — dense operators for n <= ~4096: φ_μ(A,c) = Σ c_k q_k(A)
                  (Prop. pro:whe-we-converge), its closed forms,
                  𝕃_μ(c) (eq:weighted_laplacian), diffusion
                  exp(-t𝕃)x0, return probability
                  (eq:average_return_probabilities), ρ(A), ρ(Z).
* ``series``    — matrix-free truncated series Σ c_k q_k v by the explicit
                  three-term recurrence for large n (the "explicit NBW
                  recurrence" of the north star).
* ``chebyshev`` — diffusion exp(-t𝕃)x0 at large n by a Chebyshev expansion on
                  the Gershgorin interval of Prop. pro:still-again-an-mmatrix.
* ``markov``    — the discrete-time chain P = I - D^{-1}𝕃 (eq:let_there_be_markov,
                  P:506-533) and its evolution p_{k+1} = p_k P.

Readings of silent/garbled passages are listed in DESIGN.md §3; each function
cites the passage it follows.  Pins (tests/test_oracle_*.py) check the oracle
against values the paper prints, closed forms, brute force and invariants.
"""

from . import coeffs, walks, dense, series, chebyshev  # noqa: F401
