"""Device path vs oracle: parity through the C ABI (pytest -m gpu).

Bar: skeleton, sepsets (serial rule), per-level edges_removed / ci_tests /
pseudo_inverses (serial-equivalent) and stop reason identical to the oracle's
Strategy::Serial run on the same correlation matrix; pseudo-inverses and
partial correlations bit-identical; z within 1e-12 relative (only log may
differ by an ulp); p-values within 1e-9 relative.
"""
import math

import numpy as np
import pytest

from tests.helpers import assert_same_result, instance, make_correlation, star_correlation

pytestmark = pytest.mark.gpu

VARIANTS = ["set", "edge"]


def cfg(pcs, strategy="set", **kw):
    return pcs.SkeletonConfig(strategy=pcs.Strategy(strategy), **kw)


@pytest.mark.parametrize("strategy", VARIANTS)
def test_star_graph_level_by_level(pcs, oracle, strategy):
    """test_skeleton.cpp:102-127."""
    c = star_correlation()
    r = pcs.run_pc_stable(c, 1000, cfg(pcs, strategy))
    assert r.edge_set() == [(0, 1), (0, 2), (0, 3)]
    assert r.levels_run() == 3
    assert r.stop_reason == pcs.StopReason.MaxDegreeReached
    assert [l.edges_removed for l in r.levels] == [1, 2, 0]
    assert r.sepsets.find(1, 2) == ()
    assert r.sepsets.find(1, 3) == (0,)
    assert r.sepsets.find(2, 3) == (0,)
    assert r.sepsets.stored_count() == 3
    assert_same_result(r, oracle.run_pc_stable(oracle.normalize_correlation(c), 1000), label="star")


def test_level_cap_and_sample_size(pcs, oracle):
    """test_skeleton.cpp:139-169."""
    c = star_correlation()
    r = pcs.run_pc_stable(c, 1000, cfg(pcs, max_level=1))
    assert r.levels_run() == 2 and r.stop_reason == pcs.StopReason.LevelCapReached
    r0 = pcs.run_pc_stable(c, 1000, cfg(pcs, max_level=0))
    assert r0.levels_run() == 1 and r0.skeleton.edge_count() == 5
    entries = [(i, j, 0.97) for i in range(5) for j in range(i + 1, 5)]
    c5 = make_correlation(5, entries)
    r5 = pcs.run_pc_stable(c5, 5, cfg(pcs))
    assert r5.stop_reason == pcs.StopReason.SampleSizeExhausted
    assert r5.levels_run() == 2
    assert [l.edges_removed for l in r5.levels] == [0, 10]
    assert r5.skeleton.edge_count() == 0
    assert_same_result(r5, oracle.run_pc_stable(oracle.normalize_correlation(c5), 5), label="m=5")


def test_level_zero_identity(pcs):
    """test_skeleton.cpp:52-68 and acceptance criterion 6 (n = 10, 100, 500)."""
    for n in (4, 10, 100, 500):
        r = pcs.run_pc_stable(np.eye(n), 1000, cfg(pcs))
        assert r.skeleton.edge_count() == 0
        assert r.levels_run() == 1
        assert r.levels[0].ci_tests == n * (n - 1) // 2
        assert r.levels[0].edges_removed == n * (n - 1) // 2
        assert r.levels[0].pseudo_inverses == 0
        assert r.sepsets.find(0, 1) == ()


def test_chain_and_collider(pcs, oracle):
    """acceptance_tests.cpp:383-425 (criterion 8) with the reference generator seeds."""
    w = np.zeros((3, 3)); w[1, 0] = 0.8; w[2, 1] = 0.9
    c = oracle.compute_correlation(oracle.sample_linear_gaussian(w, 10000, 31))
    r = pcs.run_pc_stable(c, 10000, cfg(pcs, alpha=0.01))
    assert r.edge_set() == [(0, 1), (1, 2)]
    assert r.sepsets.find(0, 2) == (1,)
    w = np.zeros((3, 3)); w[2, 0] = 0.8; w[2, 1] = 0.9
    c = oracle.compute_correlation(oracle.sample_linear_gaussian(w, 10000, 32))
    r = pcs.run_pc_stable(c, 10000, cfg(pcs, alpha=0.01))
    assert r.edge_set() == [(0, 2), (1, 2)]
    assert r.sepsets.find(0, 1) == ()


@pytest.mark.parametrize("strategy", VARIANTS)
def test_strategy_equivalence_instances(pcs, oracle, strategy):
    """acceptance criterion 1 instances (acceptance_tests.cpp:118-159), full serial parity."""
    for inst in range(50):
        p = (20, 50, 100)[inst % 3]
        d = (0.1, 0.2, 0.3)[(inst // 3) % 3]
        seed = 1000 + inst
        c = instance(oracle, p, d, 1000, seed)
        ref = oracle.run_pc_stable(c, 1000, alpha=0.05, strategy=oracle.KEYS, workers=8)
        dev = pcs.run_pc_stable(c, 1000, cfg(pcs, strategy, alpha=0.05))
        assert_same_result(dev, ref, label=f"inst {inst} {strategy}")


@pytest.mark.parametrize("strategy", VARIANTS)
def test_config_c1(pcs, oracle, strategy):
    """BASELINE config C1: p=100, m=1000, E[deg]=2, alpha=0.01 (bench seed 0)."""
    c = instance(oracle, 100, 2.0 / 99.0, 1000, 0)
    ref = oracle.run_pc_stable(c, 1000, alpha=0.01)  # Strategy::Serial, the sepset oracle
    dev = pcs.run_pc_stable(c, 1000, cfg(pcs, strategy, alpha=0.01))
    assert_same_result(dev, ref, label="C1")


def test_dense_deep_levels(pcs, oracle):
    """Denser graphs reach levels 3..6: exercises the templated pinv for larger ell."""
    for seed, (p, d, m) in enumerate([(40, 0.5, 300), (60, 0.4, 500), (30, 0.7, 200)]):
        c = instance(oracle, p, d, m, 77 + seed)
        ref = oracle.run_pc_stable(c, m, alpha=0.05, strategy=oracle.KEYS, workers=8)
        for strategy in VARIANTS:
            dev = pcs.run_pc_stable(c, m, cfg(pcs, strategy, alpha=0.05))
            assert_same_result(dev, ref, label=f"deep {p},{d},{m} {strategy}")


def _random_blocks(rng, ell, n):
    out = []
    for t in range(n):
        kind = t % 4
        if kind == 0:   # SPD Gram
            x = rng.normal(size=(ell + 10, ell))
            a = x.T @ x / (ell + 10)
        elif kind == 1:  # correlation block with a duplicated variable (rank deficient)
            x = rng.normal(size=(ell + 10, ell))
            if ell >= 2:
                x[:, -1] = x[:, 0]
            a = np.corrcoef(x, rowvar=False) if ell > 1 else np.ones((1, 1))
        elif kind == 2:  # exact low rank
            r = (ell + 1) // 2
            a = rng.normal(size=(ell, r)) @ rng.normal(size=(r, ell))
        else:           # near-collinear correlation block
            x = rng.normal(size=(50, ell))
            x[:, :] += 3.0 * rng.normal(size=(50, 1))
            a = np.corrcoef(x, rowvar=False) if ell > 1 else np.ones((1, 1))
        out.append(np.atleast_2d(a))
    return np.stack(out)


@pytest.mark.parametrize("ell", list(range(1, 17)) + [24, 40])
def test_pseudo_inverse_bitwise(pcs, oracle, ell):
    rng = np.random.default_rng(ell)
    a = _random_blocks(rng, ell, 64)
    got = pcs.pseudo_inverse_batch(a)
    want = np.stack([oracle.pseudo_inverse(x) for x in a])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), "device pinv differs from oracle"


def test_pseudo_inverse_pinned(pcs):
    """test_stats.cpp:178-190."""
    assert np.allclose(pcs.pseudo_inverse_batch(np.eye(4))[0], np.eye(4), atol=1e-12)
    assert np.allclose(pcs.pseudo_inverse_batch(np.diag([2.0, 4.0]))[0], np.diag([0.5, 0.25]), atol=1e-12)
    assert np.allclose(pcs.pseudo_inverse_batch(np.ones((2, 2)))[0], np.full((2, 2), 0.25), atol=1e-10)
    assert not pcs.pseudo_inverse_batch(np.zeros((3, 3)))[0].any()


@pytest.mark.parametrize("ell", list(range(0, 13)) + [20])
def test_ci_test_batch_vs_oracle(pcs, oracle, ell):
    """z within 1e-12 relative, rho and decisions identical, p-values within 1e-9 relative."""
    rng = np.random.default_rng(100 + ell)
    p = 40
    c = instance(oracle, p, 0.3, 200, 500 + ell)
    n = 400
    ij, sets = [], []
    for _ in range(n):
        pick = rng.choice(p, size=ell + 2, replace=False)
        ij.append(pick[:2])
        sets.append(np.sort(pick[2:]))
    ij = np.array(ij, np.int32)
    sets = np.array(sets, np.int32).reshape(n, ell)
    m = 200
    tau = oracle.threshold_tau(0.05, m, ell)
    ind, z, rho, deg = pcs.ci_test_batch(c, ell, ij, sets, tau)
    dof = m - ell - 3
    for k in range(n):
        wi, wz, wrho, wdeg = oracle.ci_test(c, int(ij[k, 0]), int(ij[k, 1]), sets[k].tolist(), tau)
        assert bool(ind[k]) == wi
        assert bool(deg[k]) == wdeg
        assert rho[k] == wrho
        if math.isinf(wz):
            assert math.isinf(z[k])
        else:
            assert abs(z[k] - wz) <= 1e-12 * max(abs(wz), 1e-300)
            pz = math.erfc(z[k] * math.sqrt(dof) / math.sqrt(2.0))
            pw = math.erfc(wz * math.sqrt(dof) / math.sqrt(2.0))
            assert abs(pz - pw) <= 1e-9 * max(pw, 1e-300) or (pz == 0.0 and pw == 0.0)


def test_degenerate_conditioning(pcs):
    """test_stats.cpp:329-336 / 364-371: duplicated variable -> dependent, z = +inf."""
    c = make_correlation(3, [(0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.5)])
    ind, z, rho, deg = pcs.ci_test_batch(c, 1, [[0, 1]], [[2]], 10.0)
    assert not ind[0] and deg[0] and math.isinf(z[0])


def test_correlation_matches_oracle(pcs, oracle):
    for (p, m, d, seed) in [(6, 200, 0.4, 11), (100, 1000, 0.02, 3), (257, 333, 0.05, 5)]:
        w = oracle.random_dag(p, d, seed)
        x = oracle.sample_linear_gaussian(w, m, seed + 1)  # (p, m) rows = variables
        want = oracle.compute_correlation(x)
        got = pcs.compute_correlation(x.T)  # (m, p) samples x variables
        assert np.max(np.abs(got - want)) < 1e-13
        assert np.array_equal(got, got.T)
        assert np.all(np.diag(got) == 1.0)


def test_correlation_errors(pcs):
    """test_stats.cpp:278-288 and DataMatrix validation (test_core.cpp:15-25)."""
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(5, 3))
    x[:, 2] = 3.25
    with pytest.raises(pcs.ZeroVarianceError) as e:
        pcs.compute_correlation(x)
    assert e.value.column == 2
    with pytest.raises(ValueError):
        pcs.compute_correlation(rng.normal(size=(3, 2)))
    bad = np.zeros((5, 3))
    bad[4, 1] = np.inf
    with pytest.raises(ValueError):
        pcs.compute_correlation(bad)


def test_bad_arguments(pcs):
    """test_skeleton.cpp:171-177 and CorrelationMatrix validation (test_core.cpp:36-51)."""
    with pytest.raises(ValueError):
        pcs.run_pc_stable(np.eye(3), 3)
    with pytest.raises(ValueError):
        pcs.run_pc_stable(np.eye(3), 100, pcs.SkeletonConfig(alpha=2.0))
    asym = np.eye(3); asym[0, 1] = 0.5; asym[1, 0] = 0.4
    with pytest.raises(ValueError):
        pcs.run_pc_stable(asym, 100)
    diag = np.eye(2); diag[1, 1] = 0.9
    with pytest.raises(ValueError):
        pcs.run_pc_stable(diag, 100)
    rng_ = np.eye(2); rng_[0, 1] = rng_[1, 0] = 1.5
    with pytest.raises(ValueError):
        pcs.run_pc_stable(rng_, 100)


def test_data_pipeline_matches(pcs, oracle):
    """run_pc_stable_data (device correlation + skeleton) agrees with the oracle on a clean instance."""
    w = oracle.random_dag(80, 0.05, 9)
    x = oracle.sample_linear_gaussian(w, 2000, 10)
    dev = pcs.run_pc_stable_data(x.T, pcs.SkeletonConfig(alpha=0.01))
    ref = oracle.run_pc_stable(oracle.compute_correlation(x), 2000, alpha=0.01)
    assert dev.edge_set() == ref.edge_set()


@pytest.mark.parametrize("variant", ["set", "edge"])
def test_run_level_chain_equals_run_pc_stable(pcs, oracle, variant):
    """pcs_run_level (run_level_zero / run_level_serial / run_level_edge_parallel / run_level_set_shared,
    skeleton.hpp:262-333) applied level by level with threshold_tau reproduces the oracle's whole run:
    same graph after every level, same sepsets, same per-level counters."""
    m, alpha = 400, 0.05
    c = instance(oracle, 40, 0.25, m, 5)
    ref = oracle.run_pc_stable(c, m, alpha=alpha)
    p = c.shape[0]
    g = np.ones((p, p), np.uint8) - np.eye(p, dtype=np.uint8)
    cfg = pcs.SkeletonConfig(alpha=alpha, strategy=pcs.Strategy(variant))
    sep = {}
    for lv in ref.levels:
        tau = oracle.threshold_tau(alpha, m, lv.level)
        g, st, removed = pcs.run_level(c, g, lv.level, tau, cfg)
        sep.update(removed)
        assert (st.level, st.ci_tests, st.edges_removed) == (lv.level, lv.ci_tests, lv.edges_removed)
    assert np.array_equal(g, ref.adjacency)
    assert sep == ref.sepsets


def test_near_threshold_tests_are_listed(pcs, oracle):
    """A level-0 pair whose |rho| sits 1e-12 (relative) either side of tanh(tau): both fall inside the
    +-1e-9 band, are decided by the exact comparison, counted and listed with their statistic; the
    decisions equal the oracle's."""
    m, alpha = 500, 0.05
    tau = oracle.threshold_tau(alpha, m, 0)
    r = math.tanh(tau)
    c = make_correlation(5, [(0, 1, r * (1 + 1e-12)), (2, 3, -r * (1 - 1e-12)), (1, 4, 0.5)])
    dev = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=alpha, max_level=0))
    ref = oracle.run_pc_stable(c, m, alpha=alpha, max_level=0)
    assert np.array_equal(dev.skeleton.cells, ref.adjacency)
    assert dev.near_threshold_count == 2 and dev.levels[0].device_near_threshold == 2
    got = sorted((x["i"], x["j"], x["independent"]) for x in dev.near_threshold)
    assert got == [(0, 1, False), (2, 3, True)]
    for x in dev.near_threshold:
        assert x["level"] == 0 and abs(abs(x["rho"]) - r) <= 2e-12 * r and abs(x["z"] - tau) < 1e-9 * tau
