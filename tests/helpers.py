"""Shared test helpers: seeded instances (reference generator semantics via the
oracle) and result comparison between the device path and the oracle."""
from __future__ import annotations

import math

import numpy as np


def instance(oracle, p: int, density: float, m: int, seed: int) -> np.ndarray:
    """random_dag(p, d, seed) + sample_linear_gaussian(dag, m, seed+1) + compute_correlation
    (bench.hpp:94-96 / acceptance_tests.cpp:129-131 convention)."""
    w = oracle.random_dag(p, density, seed)
    x = oracle.sample_linear_gaussian(w, m, seed + 1)
    return oracle.compute_correlation(x, threads=8)


def make_correlation(n: int, entries) -> np.ndarray:
    """support.hpp:103-111."""
    c = np.eye(n)
    for i, j, v in entries:
        c[i, j] = c[j, i] = v
    return c


def star_correlation() -> np.ndarray:
    """test_skeleton.cpp:27-32."""
    s = 1.0 / math.sqrt(3.0)
    t = math.sqrt(3.0) / 2.0
    return make_correlation(4, [(0, 1, s), (0, 2, s), (0, 3, t), (1, 2, 0.0), (1, 3, 0.5), (2, 3, 0.5)])


def assert_same_result(dev, ref, counters: bool = True, label: str = ""):
    """Device SkeletonResult vs oracle SkeletonResult (serial strategy)."""
    assert np.array_equal(dev.skeleton.cells, ref.adjacency), f"{label}: skeleton differs"
    assert dev.stop_reason.value == ref.stop_reason, f"{label}: stop reason {dev.stop_reason} vs {ref.stop_reason}"
    assert dev.levels_run() == ref.levels_run(), f"{label}: levels {dev.levels_run()} vs {ref.levels_run()}"
    got = dev.sepsets.as_dict()
    assert got == ref.sepsets, f"{label}: sepsets differ"
    for a, b in zip(dev.levels, ref.levels):
        assert a.level == b.level
        assert a.edges_removed == b.edges_removed, f"{label}: level {a.level} removed {a.edges_removed} vs {b.edges_removed}"
        if counters:
            assert a.ci_tests == b.ci_tests, f"{label}: level {a.level} ci_tests {a.ci_tests} vs {b.ci_tests}"
            assert a.pseudo_inverses == b.pseudo_inverses, f"{label}: level {a.level} pinv"
