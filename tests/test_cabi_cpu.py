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
    assert (o.krylov_dim, o.reorth, o.max_cols, o.breakdown_tol, o.rho_bound, o.relabel) == (30, 1, 32, 1e-12, 0.0, 1)
    assert (o.solver, o.cg_tol, o.cg_maxit, o.cg_check) == (0, 1e-9, 1000, 8)


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
