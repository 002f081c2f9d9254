"""CPU checks of bench.py's host logic: the algorithmic-bytes model behind every `roofline` and the
JSON contract helpers.  No GPU: bench.py is imported, not run."""
import importlib.util
import os

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


C4 = dict(n=10_000_000, nnz=400_000_000, n_halo=0, G=11, K=30, Bmax=11, b=1, n_theta=11)


def test_c4_spmv_bytes_match_the_survey_formula(bench):
    """per Z-step 4 nnz + 4(n+1) + 8nB (y) + 8nB (x) + 8nB (out); plus the two b = 1 seeds."""
    ab = bench.algorithmic_bytes(**C4)
    n, nnz, B, K = C4["n"], C4["nnz"], 11, 30
    csr = 4 * nnz + 4 * (n + 1)
    z_step = csr + 3 * 8 * n * B
    seeds = 2 * (csr + 2 * 8 * n * 1)
    assert ab["spmv_binned"] == K * z_step + seeds
    # per launch (32 launches) ≈ 4.125 GB, the DESIGN §7 figure
    assert abs(ab["spmv_binned"] / 32 / 1e9 - 4.125) < 0.01


def test_toar_gram_bytes(bench):
    """TOAR step j: the dot pass reads j + 3 n x B blocks, the update pass reads j + 3 and writes 3."""
    ab = bench.algorithmic_bytes(**C4)
    blk = 8 * C4["n"] * 11
    K = 30
    assert ab["dcgs2_dots"] == 2 * blk + sum((j + 3) * blk for j in range(K)) + (K + 2) * blk
    assert ab["toar_update"] == 3 * blk + sum((j + 6) * blk for j in range(K))


def test_fp32_and_active_rows_scale_the_batch_blocks(bench):
    """fp32 storage halves every stored block of the batch (not the double seeds, inputs, outputs); the active rows
    (wl_operator_active_rows) shrink the batch's blocks but not the outputs."""
    f64 = bench.algorithmic_bytes(**C4)
    f32 = bench.algorithmic_bytes(**C4, esz=4)
    assert f32["dcgs2_dots"] * 2 == f64["dcgs2_dots"] and f32["toar_update"] * 2 == f64["toar_update"]
    assert f64["spmv_binned"] / 2 < f32["spmv_binned"] < f64["spmv_binned"]   # col ids and seeds stay
    na = 6_000_000
    act = bench.algorithmic_bytes(**C4, n_act=na)
    assert act["dcgs2_dots"] * C4["n"] == f64["dcgs2_dots"] * na
    out = 8 * C4["n"] * 11 + 8 * C4["n"] * 1 + 8 * C4["n"] * 11   # combine: output, V, t' over all rows
    assert act["combine"] == 32 * 8 * na * 11 + out


def test_dcgs2_bytes(bench):
    ab = bench.algorithmic_bytes(**C4, reorth=1)
    vec = 8 * 2 * C4["n"] * 11
    K = 30
    assert ab["dcgs2_dots"] == sum((j + 1.5) * vec for j in range(K)) + (K + 1) * vec
    assert ab["dcgs2_update"] == sum((j + 3.5) * vec for j in range(K))
