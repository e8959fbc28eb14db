"""Parity at the BASELINE configs' full sizes beyond C1/C2 (tests/test_gpu_parity.py,
tests/test_gpu_c2_sampled.py), with one correlation matrix (the oracle's bits) fed to both sides:

  * C3 (DREAM5 shape, p=1643, m=850, d=0.01) and C4 (S.cerevisiae shape, p=5361, m=63, d=0.002):
    the whole run -- skeleton, serial-rule sepsets, per-level counters, stop reason -- identical to
    the oracle's (Strategy::Serial semantics, computed in the oracle's parallel key mode);
  * C5 (scaling sweep point p=5000, m=5000, d=0.05, rescaled generator): level 0 in full and level 1
    on samples of the device's snapshot (the oracle's level-1 keys for the sampled edges), since the
    oracle cannot run level 1's 7.7e10 serial tests in test time.
Seeds follow bench.hpp:94-96 (7919 x config index)."""
import os
import time

import numpy as np
import pytest

from tests.helpers import assert_same_result, instance
from tests.test_gpu_c2_sampled import NONE, _device_keys, _full_row_keys

pytestmark = pytest.mark.gpu
THREADS = max(1, min(16, os.cpu_count() or 1))


@pytest.mark.parametrize("name,p,d,m,seed", [("C3", 1643, 0.01, 850, 2 * 7919), ("C4", 5361, 0.002, 63, 3 * 7919)])
def test_full_config_matches_oracle(pcs, oracle, name, p, d, m, seed):
    c = instance(oracle, p, d, m, seed)
    ref = oracle.run_pc_stable(c, m, alpha=0.01, strategy=oracle.KEYS, workers=THREADS)
    for variant in ("set", "edge"):
        dev = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=0.01, strategy=pcs.Strategy(variant)))
        assert_same_result(dev, ref, label=f"{name} {variant}")


def test_c5_level0_full_level1_sampled(pcs, oracle):
    p, m, d, seed, alpha = 5000, 5000, 0.05, 4 * 7919, 0.01
    w = pcs.random_dag(p, d, seed)
    x, _ = pcs.sample_linear_gaussian_rescaled(w, m, seed + 1)
    del w
    c = oracle.compute_correlation(np.ascontiguousarray(x.T), threads=THREADS)
    del x
    ref0 = oracle.run_pc_stable(c, m, alpha=alpha, max_level=0, strategy=oracle.KEYS, workers=THREADS)
    s = pcs.Session(c, m, pcs.SkeletonConfig(alpha=alpha, max_level=1))
    try:
        running, ell, _ = s.level_begin()
        assert running and ell == 0
        s.level_pass(0)
        s.level_pass(1)
        s.level_end()
        running, ell, n = s.level_begin()
        assert running and ell == 1
        off, idx = s.snapshot(p)
        # the level-1 snapshot is the level-0 skeleton: identical to the oracle's
        adj = np.zeros((p, p), np.uint8)
        rows = np.repeat(np.arange(p), np.diff(off))
        adj[rows, idx] = 1
        assert np.array_equal(adj, ref0.adjacency), "C5 level-0 skeleton"
        s.level_pass(0)
        s.level_pass(1)
        ptr, n = s.keys()
        keys = _device_keys(ptr, n)
        tau = oracle.threshold_tau(alpha, m, 1)
        a, b = rows[idx > rows], idx[idx > rows]
        starts = np.linspace(0, n - 64, 32).astype(int)
        nchk, nrem, t0 = 0, 0, time.time()
        for st in starts:
            e1 = int(st) + 48
            refk = oracle.level_keys(c, off, idx, 1, tau, int(st), e1, threads=THREADS)
            refk = _full_row_keys(oracle, refk, int(st), a, b, off, idx, 1)
            got = keys[st:e1]
            bad = np.nonzero(refk != got)[0]
            assert len(bad) == 0, f"C5 level 1 edges {st + bad[:5]}: device {got[bad[:5]]} oracle {refk[bad[:5]]}"
            nchk += e1 - int(st)
            nrem += int((refk != NONE).sum())
        s.level_end()
        res = s.finish(with_sepsets=False)
    finally:
        s.close()
    assert res.levels[0].edges_removed == ref0.levels[0].edges_removed
    assert nchk >= 1000 and nrem > 0, (nchk, nrem)
    print(f"C5: level-1 keys checked on {nchk} edges ({nrem} removed) in {time.time() - t0:.1f}s")
