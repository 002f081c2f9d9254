"""CPU-only checks of the C ABI boundary: the library loads, exports every symbol
include/walklap.h declares, and its host-side logic (partition, options) is exact."""
import ctypes
import os
import re

import numpy as np
import pytest

import graphgen as gg
from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2601_11338_b200 import build
    build.build()
    import paper_2601_11338_b200 as wl
    return wl.load()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "walklap.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wl_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = declared_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name


def test_opts_default(lib):
    import paper_2601_11338_b200.walklap as w
    o = w._Opts()
    lib.wl_opts_default(ctypes.byref(o))
    assert (o.krylov_dim, o.reorth, o.max_cols, o.breakdown_tol, o.rho_bound, o.relabel) == (30, 2, 32, 1e-12, 0.0, 1)
    assert (o.solver, o.cg_tol, o.cg_maxit, o.cg_check, o.tol) == (0, 1e-9, 1000, 8, 0.0)
    assert (o.halo_overlap, o.lanczos, o.krylov_adaptive, o.fp32) == (1, 1, 0, 0)


def _partition_def(row_ptr, P):
    """Definition from walklap.h: bounds[p] = smallest r with row_ptr[r] >= ceil(p*nnz/P)."""
    nnz = int(row_ptr[-1] - row_ptr[0])
    out = [0]
    for p in range(1, P):
        target = row_ptr[0] + -(-p * nnz // P)
        r = int(np.searchsorted(row_ptr, target, side="left"))
        out.append(min(max(r, out[-1]), len(row_ptr) - 1))
    out.append(len(row_ptr) - 1)
    return np.array(out)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_is_exact_and_balanced(lib, P):
    import paper_2601_11338_b200 as wl
    for g in (gg.rmat(14, 12000, 100000, seed=1, perm_seed=2), gg.barabasi_albert(5000, 3, 1), gg.path(5)):
        b = wl.partition(g.row_ptr, P)
        assert np.array_equal(b, _partition_def(g.row_ptr, P))
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
        nnz = np.diff(g.row_ptr[b])
        assert nnz.max() <= g.nnz / P + g.degrees.max() + 1


def test_no_cpu_fallback_in_product(lib):
    """The product package never imports the oracle and has no numpy compute path."""
    pkg = os.path.join(ROOT, "paper_2601_11338_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("# oracle", ""), fn
            assert "scipy" not in src, fn


def _hessenberg(rng, n, kind):
    H = np.triu(rng.standard_normal((n, n)), -1)
    if kind == "companion":  # roots of a random polynomial: many complex pairs
        H = np.zeros((n, n))
        H[0, :] = rng.standard_normal(n)
        H[np.arange(1, n), np.arange(n - 1)] = 1.0
    elif kind == "deflated":  # exact zeros on the subdiagonal
        H[np.arange(1, n, 3), np.arange(0, n - 1, 3)] = 0.0
    elif kind == "symmetric":  # tridiagonal symmetric: real spectrum
        d, e = rng.standard_normal(n), rng.standard_normal(n - 1)
        H = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    return H


@pytest.mark.parametrize("kind", ["random", "companion", "deflated", "symmetric"])
def test_hessenberg_eigvals_match_lapack(lib, kind):
    """The host Francis QR behind wl_spectral_radius_z (eig.cu) against LAPACK (numpy.linalg.eigvals),
    as multisets, for sizes 1..64 — including complex pairs, exact deflations and real spectra."""
    import paper_2601_11338_b200 as wl
    rng = np.random.default_rng(7)
    for n in list(range(1, 13)) + [20, 31, 48, 64]:
        H = _hessenberg(rng, n, kind)
        got = wl.hessenberg_eigvals(H)
        ref = np.linalg.eigvals(H)
        scale = max(1.0, np.abs(ref).max())
        # greedy matching (multisets)
        left = list(ref)
        for z in got:
            k = int(np.argmin([abs(z - r) for r in left]))
            assert abs(z - left[k]) <= 1e-8 * scale, (kind, n, z, left[k])
            left.pop(k)


def test_hessenberg_eigvals_closed_forms(lib):
    import paper_2601_11338_b200 as wl
    # rotation generator: ±i; Jordan-like upper triangular: its diagonal; 2x2 real pair
    assert np.allclose(sorted(wl.hessenberg_eigvals(np.array([[0.0, -1.0], [1.0, 0.0]])), key=lambda z: z.imag), [-1j, 1j])
    T = np.triu(np.arange(1.0, 26.0).reshape(5, 5))
    assert np.allclose(np.sort(wl.hessenberg_eigvals(T).real), [1.0, 7.0, 13.0, 19.0, 25.0])
    assert np.allclose(np.sort(wl.hessenberg_eigvals(np.array([[2.0, 1.0], [1.0, 2.0]])).real), [1.0, 3.0])


@pytest.mark.parametrize("method", [0, 1])
def test_symmetric_eig_matches_lapack(lib, method):
    """The host eigensolvers behind wl_xnystrace_exp (trace.cu) against LAPACK (numpy.linalg.eigh):
    eigenvalues, residual ‖A z − λ z‖ and orthonormality, including repeated eigenvalues."""
    import paper_2601_11338_b200 as wl
    rng = np.random.default_rng(3)
    for n in [1, 2, 3, 7, 24, 61, 130]:
        G = rng.standard_normal((n, n))
        Qr = np.linalg.qr(rng.standard_normal((n, n)))[0]
        for A in (G + G.T, (Qr * np.resize([1.0, 1.0, 2.0, 2.0], n)) @ Qr.T):
            lam, Z = wl.symmetric_eig(A, method)
            assert np.allclose(np.sort(lam), np.linalg.eigvalsh(A), atol=1e-12 * max(1, np.abs(A).max()))
            assert np.abs(A @ Z - Z * lam).max() <= 1e-12 * max(1, np.abs(A).max()) * n
            assert np.abs(Z.T @ Z - np.eye(n)).max() <= 1e-12 * n


def test_xnystrace_curve_matches_oracle(lib):
    """The host estimator behind wl_xnystrace_exp against oracle/trace.xnystrace, with exact Y(t):
    the projected space is the whole space (d = n) and lam, Q come from LAPACK."""
    import paper_2601_11338_b200 as wl
    import scipy.linalg as sla
    import graphgen as gg
    from oracle import dense as D
    from oracle import trace as T
    L = D.standard_laplacian(D.adjacency(gg.karate()))
    lam, Q = np.linalg.eigh(L)
    ts = np.linspace(0.0, 10.0, 30)
    for M in (1, 2, 5, 12):
        Om = gg.vectors(34, M, 40 + M)
        p, e = wl.xnystrace_curve(lam, Q.T @ Om, 34, ts)
        ref = np.array([T.xnystrace(sla.expm(-t * L) @ Om / 34, Om) for t in ts])
        assert np.max(np.abs(p - ref[:, 0]) / np.abs(ref[:, 0])) < 1e-9, M
        assert np.max(np.abs(e - ref[:, 1])) <= 1e-9 * np.max(ref[:, 0]) + 1e-7 * np.max(ref[:, 1]), M


def test_aaa_exp_poles_host_routine(lib):
    """wl_aaa_exp_poles (host, no GPU): the library's AAA poles carry a rational approximation of exp(-x) on
    [0, X] as good as the oracle's (least-squares fit over the poles on the sample set, ~1e-13).  The poles
    themselves may differ from the oracle's: AAA's null vector of a Loewner matrix with a tiny singular gap is
    method dependent, so GPU parity tests pass the SAME poles to both sides."""
    import paper_2601_11338_b200 as wl
    from oracle import aaa as AA
    for X in (10.0, 100.0, 1000.0, 30.5):
        p = wl.aaa_exp_poles(X)
        Z = np.concatenate([[0.0], X * np.logspace(-10.0, 0.0, 2000)])
        allp = [q for x in p for q in ((x, np.conj(x)) if x.imag != 0 else (x,))]
        B = np.column_stack([np.ones_like(Z)] + [1.0 / (Z - q) for q in allp]).astype(complex)
        c, *_ = np.linalg.lstsq(B, np.exp(-Z).astype(complex), rcond=None)
        assert np.abs(B @ c - np.exp(-Z)).max() < 1e-12, X
        assert np.all(p.imag >= 0) and abs(len(p) - len(AA.exp_poles(X))) <= 1
