"""The oracle's set-shared serial-key mode (ORC_FAST) and its device-order correlation, which make the
whole-run golden fixtures (tests/golden/*_full.npz, tools/make_golden.py) -- CPU only.

* ORC_FAST is result-identical to Strategy::Serial (skeleton.hpp:292-307): skeleton, serial-rule
  sepsets, per-level ci_tests / pseudo_inverses / edges_removed, stop reason -- checked against the
  plain serial restatement on many small seeded instances, dense enough to reach deep levels (l > 4
  takes the scalar path) and both edge directions.
* compute_correlation_fma (tree means + FMA-chain Gram, the device's pinned order) agrees with the
  reference-order restatement to rounding, and is symmetric with a unit diagonal.
* The committed fixtures of the small configs regenerate bit for bit (digests, per-row hashes,
  counters), so the fixture pipeline itself is deterministic."""
import os

import numpy as np
import pytest

from tests.golden_tools import canon_from_oracle, compare
from tests.helpers import instance

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same(a, b):
    assert np.array_equal(a.adjacency, b.adjacency)
    assert a.sepsets == b.sepsets
    assert [(l.ci_tests, l.pseudo_inverses, l.edges_removed) for l in a.levels] == \
        [(l.ci_tests, l.pseudo_inverses, l.edges_removed) for l in b.levels]
    assert a.stop_reason == b.stop_reason


@pytest.mark.parametrize("shape", [(20, 0.3, 50), (30, 0.5, 200), (40, 0.2, 30), (60, 0.15, 100), (25, 0.6, 40)])
def test_fast_equals_serial(oracle, shape):
    p, d, m = shape
    for seed in range(12):
        c = instance(oracle, p, d, m, 7 * seed + 1)
        fast = oracle.run_pc_stable(c, m, alpha=0.05, strategy=oracle.FAST, workers=3)
        ser = oracle.run_pc_stable(c, m, alpha=0.05, strategy=oracle.SERIAL)
        _same(fast, ser)


def test_fast_level_keys_match_per_test_keys(oracle):
    """orc_level_keys_fast == orc_level_keys (per-test pseudo-inverse) on a level-2 snapshot."""
    c = instance(oracle, 80, 0.2, 300, 11)
    r = oracle.run_pc_stable(c, 300, alpha=0.05, strategy=oracle.SERIAL, max_level=1)
    adj = r.adjacency.astype(bool)
    off = np.concatenate([[0], np.cumsum(adj.sum(1))]).astype(np.int32)
    idx = np.nonzero(adj)[1].astype(np.int32)
    tau = oracle.threshold_tau(0.05, 300, 2)
    a = oracle.level_keys(c, off, idx, 2, tau, threads=2)
    b = oracle.level_keys_fast(c, off, idx, 2, tau, threads=2)
    assert np.array_equal(a, b)
    assert (a != oracle.NONE_KEY).any()


def test_fma_correlation_close_to_reference_order(oracle):
    w = oracle.random_dag(120, 0.05, 5)
    x = oracle.sample_linear_gaussian(w, 700, 6)
    cf = oracle.compute_correlation_fma(x, threads=4)
    cs = oracle.compute_correlation(x, threads=4)
    assert np.array_equal(cf, cf.T) and np.all(np.diag(cf) == 1.0)
    assert np.abs(cf - cs).max() < 1e-13


@pytest.mark.parametrize("name", ["C1", "C3", "C4"])
def test_small_fixtures_regenerate(oracle, name):
    import hashlib

    from tools.make_golden import ALPHA, CASES, case_data

    path = os.path.join(GOLD, f"{name.lower()}_full.npz")
    g = dict(np.load(path))
    x, xsha = case_data(name)
    assert xsha == str(g["data_sha256"])
    c = oracle.compute_correlation_fma(x, threads=8)
    assert hashlib.sha256(c.tobytes()).hexdigest() == str(g["corr_sha256"])
    ml = CASES[name][4]
    r = oracle.run_pc_stable_arrays(c, int(g["m"]), alpha=ALPHA, max_level=ml, strategy=oracle.FAST, workers=8)
    assert compare(canon_from_oracle(r), g) == []
