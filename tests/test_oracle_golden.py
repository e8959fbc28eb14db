"""Pins the CPU oracle (oracle/pcs_oracle.c) against every known-answer test and
golden value the reference's own suite holds for the hot path
(proj/tests/test_stats.cpp, test_comb.cpp, test_core.cpp, test_skeleton.cpp,
acceptance_tests.cpp).  The reference itself cannot be built here (no Eigen3 /
GoogleTest), so these pins are what make the oracle trustworthy."""
import itertools
import math

import numpy as np
import pytest

from tests.helpers import instance, make_correlation, star_correlation


# ------------------------------------------------------------------ stats
def test_normal_quantile_known_values(oracle):  # test_stats.cpp:21-27
    assert oracle.normal_quantile(0.5) == 0.0
    assert abs(oracle.normal_quantile(0.975) - 1.9599639845400545) <= 1e-13
    assert abs(oracle.normal_quantile(0.995) - 2.5758293035489004) <= 1e-13
    assert abs(oracle.normal_quantile(0.841344746068543) - 1.0) <= 1e-12
    assert abs(oracle.normal_quantile(0.022750131948179195) + 2.0) <= 1e-12


def test_normal_quantile_round_trip_and_domain(oracle):  # test_stats.cpp:29-43
    p = 1e-10
    while p < 1.0:
        q = oracle.normal_quantile(p)
        assert abs(0.5 * math.erfc(-q / math.sqrt(2.0)) / p - 1.0) <= 1e-9
        p = p * 3.7 if p < 0.5 else 1.0 - (1.0 - p) / 3.7
    for p in (0.9, 0.99, 0.999, 0.6, 0.51):
        assert abs(oracle.normal_quantile(p) + oracle.normal_quantile(1.0 - p)) <= 1e-13
    for bad in (0.0, 1.0, -0.3):
        with pytest.raises(oracle.OracleError):
            oracle.normal_quantile(bad)


def test_fisher_z(oracle):  # test_stats.cpp:45-58
    assert oracle.fisher_z(0.0) == 0.0
    assert abs(oracle.fisher_z(0.5) - 0.5493061443340549) <= 1e-15
    assert abs(oracle.fisher_z(0.9) - 1.4722194895832204) <= 1e-15
    # EXPECT_DOUBLE_EQ: within 4 ulps
    assert abs(oracle.fisher_z(0.7) - oracle.fisher_z(-0.7)) <= 4 * np.spacing(oracle.fisher_z(0.7))
    prev = -1.0
    for k in range(100):
        z = oracle.fisher_z(k * 0.01)
        assert z > prev
        prev = z
    for bad in (1.0, -1.0, float("nan")):
        with pytest.raises(oracle.OracleError):
            oracle.fisher_z(bad)


def test_threshold_tau(oracle):  # test_stats.cpp:60-80
    tau = oracle.threshold_tau(0.05, 1000, 0)
    assert abs(tau - 0.062073) <= 1e-6
    assert tau == oracle.normal_quantile(0.975) / math.sqrt(997.0)
    assert oracle.threshold_tau(1.0 - 1e-16, 100, 0) >= 0.0
    assert oracle.threshold_tau(0.05, 2000, 0) < oracle.threshold_tau(0.05, 1000, 0)
    assert oracle.threshold_tau(0.05, 1000, 0) < oracle.threshold_tau(0.05, 1000, 1)
    assert oracle.threshold_tau(0.05, 1000, 3) < oracle.threshold_tau(0.01, 1000, 3)
    oracle.threshold_tau(0.05, 8, 4)
    for args, code in [((0.05, 7, 4), oracle.ELEVEL), ((0.05, 4, 1), oracle.ELEVEL), ((0.0, 100, 0), oracle.EINVAL),
                       ((1.1, 100, 0), oracle.EINVAL), ((0.05, 100, -1), oracle.EINVAL)]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.threshold_tau(*args)
        assert e.value.code == code


def test_tau_alpha_one_is_zero(oracle):  # test_stats.cpp:63-64 (alpha = 1 allowed, stats.hpp:121)
    assert oracle.threshold_tau(1.0, 100, 0) == 0.0


def test_correlation_perfect_and_direct_formula(oracle):  # test_stats.cpp:81-106
    x = np.array([[1, 2, 3, 4, 5, 6]], float)
    data = np.vstack([x, x, -x])
    c = oracle.compute_correlation(data)
    assert c[0, 1] == 1.0 and c[0, 2] == -1.0 and c[0, 0] == 1.0
    w = oracle.random_dag(6, 0.4, 11)
    xs = oracle.sample_linear_gaussian(w, 200, 12)
    c = oracle.compute_correlation(xs)
    for i in range(6):
        for j in range(6):
            a = xs[i] - xs[i].mean()
            b = xs[j] - xs[j].mean()
            assert abs(c[i, j] - a @ b / math.sqrt((a @ a) * (b @ b))) <= 1e-14


def test_correlation_zero_variance_column(oracle):  # test_stats.cpp:108-117
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, size=(3, 5))
    x[2] = 3.25
    with pytest.raises(oracle.OracleError) as e:
        oracle.compute_correlation(x)
    assert e.value.code == oracle.EZEROVAR and e.value.column == 2


def test_correlation_matrix_validation(oracle):  # test_core.cpp:27-57
    c = np.array([[1.0 + 5e-13, 0.5 + 4e-13], [0.5, 1.0]])
    n = oracle.normalize_correlation(c)
    assert n[0, 0] == 1.0 and n[0, 1] == n[1, 0] and abs(n[0, 1] - 0.5) <= 1e-12
    c = np.eye(2); c[0, 1] = c[1, 0] = 1.0 + 5e-13
    assert oracle.normalize_correlation(c)[0, 1] == 1.0
    bad = [np.eye(3), np.eye(2), np.eye(2)]
    bad[0][0, 1] = 0.5; bad[0][1, 0] = 0.4
    bad[1][1, 1] = 0.9
    bad[2][0, 1] = bad[2][1, 0] = 1.5
    for b in bad:
        with pytest.raises(oracle.OracleError):
            oracle.normalize_correlation(b)


# ------------------------------------------------------------------ comb
def test_binomials(oracle):  # test_comb.cpp:13-45
    assert oracle.binomial(5, 2) == 10 and oracle.binomial(6, 2) == 15
    assert oracle.binomial(0, 0) == 1 and oracle.binomial(7, 0) == 1 and oracle.binomial(7, 7) == 1
    assert oracle.binomial(64, 32) == 1832624140942590534
    for n in range(65):
        for k in range(n + 1):
            assert oracle.binomial(n, k) == math.comb(n, k)
    assert oracle.binomial(65, 1) == 65 and oracle.binomial(65, 2) == 2080
    assert oracle.binomial(100, 3) == 161700 and oracle.binomial(200, 5) == 2535650040
    assert oracle.binomial(1000, 2) == 499500
    for args in ((-1, 0), (3, 4), (3, -1)):
        with pytest.raises(oracle.OracleError) as e:
            oracle.binomial(*args)
        assert e.value.code == oracle.EINVAL
    with pytest.raises(oracle.OracleError) as e:
        oracle.binomial(200, 100)
    assert e.value.code == oracle.EOVERFLOW


def test_unrank_pins(oracle):  # test_comb.cpp:47-54, 78-88
    one = lambda n, l, t: [v + 1 for v in oracle.unrank_positions(n, l, t)]
    assert one(3, 2, 0) == [1, 2] and one(3, 2, 1) == [1, 3] and one(3, 2, 2) == [2, 3]
    assert one(5, 5, 0) == [1, 2, 3, 4, 5]
    assert oracle.unrank_positions(6, 2, 0) == [0, 1] and oracle.unrank_positions(6, 2, 14) == [4, 5]
    assert oracle.unrank_positions_excluding(5, 2, 9, 4) == [3, 5]  # the paper's Fig. 5 example
    assert oracle.unrank_positions_excluding(1, 1, 0, 0) == [1]
    for args in ((5, 2, 10), (3, 4, 0)):
        with pytest.raises(oracle.OracleError):
            oracle.unrank_positions(*args)


def _rank_of(n, combo_1based):  # support.hpp:44-54 (Eq. 2)
    ell = len(combo_1based)
    t, prev = 0, 0
    for c in range(ell):
        for k in range(prev + 1, combo_1based[c]):
            t += math.comb(n - k, ell - (c + 1))
        prev = combo_1based[c]
    return t


def test_unranking_exhaustive(oracle):  # acceptance criterion 2 (acceptance_tests.cpp:164-187)
    checked = 0
    for width in range(0, 17):
        for ell in range(0, 7):
            if ell > width:
                continue
            for t, combo in enumerate(itertools.combinations(range(width), ell)):
                got = oracle.unrank_positions(width, ell, t)
                assert got == list(combo)
                assert _rank_of(width, [v + 1 for v in got]) == t
                checked += 1
    assert checked > 20000


def test_exclusion_unranking(oracle):  # acceptance criterion 3 (acceptance_tests.cpp:191-217)
    for row_width in range(1, 13):
        for ell in range(0, min(4, row_width - 1) + 1):
            for skip in range(row_width):
                want = [list(c) for c in itertools.combinations(range(row_width), ell) if skip not in c]
                assert len(want) == math.comb(row_width - 1, ell)
                for t, combo in enumerate(want):
                    assert oracle.unrank_positions_excluding(row_width - 1, ell, t, skip) == combo


def test_next_combination(oracle):  # test_comb.cpp:117-131
    for n in range(1, 10):
        for ell in range(1, n + 1):
            cur = oracle.unrank_positions(n, ell, 0)
            total = math.comb(n, ell)
            for t in range(1, total):
                ok, cur = oracle.next_combination(cur, n)
                assert ok and cur == oracle.unrank_positions(n, ell, t)
            ok, last = oracle.next_combination(cur, n)
            assert not ok and last == cur


# ------------------------------------------------------------------ pseudo-inverse / partial correlation
def test_pinv_pinned(oracle):  # test_stats.cpp:178-190
    assert np.allclose(oracle.pseudo_inverse(np.eye(4)), np.eye(4), atol=1e-12)
    assert np.allclose(oracle.pseudo_inverse(np.diag([2.0, 4.0])), np.diag([0.5, 0.25]), atol=1e-12)
    assert np.allclose(oracle.pseudo_inverse(np.ones((2, 2))), np.full((2, 2), 0.25), atol=1e-10)
    assert not oracle.pseudo_inverse(np.zeros((3, 3))).any()
    with pytest.raises(oracle.OracleError):
        oracle.pseudo_inverse(np.zeros((2, 3)))
    nan = np.zeros((2, 2)); nan[0, 0] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.pseudo_inverse(nan)


def test_pinv_penrose_conditions(oracle):  # acceptance criterion 5 (acceptance_tests.cpp:268-326)
    rng = np.random.default_rng(60000)
    for idx in range(500):
        ell = 1 + idx % 14
        kind = (idx // 14) % 4
        invertible = False
        if idx == 0:
            a = np.zeros((5, 5))
        elif kind == 0:
            x = rng.normal(size=(ell + 10, ell)); a = x.T @ x / (ell + 10); invertible = True
        elif kind == 1:
            a = rng.normal(size=(ell, ell)) + (4.0 + 2.0 * math.sqrt(ell)) * np.eye(ell); invertible = True
        elif kind == 2:
            r = (ell + 1) // 2
            a = rng.normal(size=(ell, r)) @ rng.normal(size=(r, ell)); invertible = r == ell
        else:
            x = rng.normal(size=(ell + 10, ell))
            if ell >= 2:
                x[:, -1] = x[:, 0]
            a = x.T @ x / (ell + 10); invertible = ell == 1
        g = oracle.pseudo_inverse(a)
        assert np.max(np.abs(a @ g @ a - a)) <= 1e-6
        assert np.max(np.abs(g @ a @ g - g)) <= 1e-6
        assert np.max(np.abs((a @ g).T - a @ g)) <= 1e-6
        assert np.max(np.abs((g @ a).T - g @ a)) <= 1e-6
        if invertible:
            assert np.max(np.abs(g - np.linalg.inv(a))) <= 1e-6


def test_pinv_matches_svd(oracle):  # test_stats.cpp:192-213 (SVD oracle of support.hpp:58-65)
    rng = np.random.default_rng(123)
    for trial in range(60):
        n = 1 + trial % 10
        a = rng.uniform(-1, 1, size=(n, n))
        if trial % 2 == 1 and n >= 2:
            r = 1 + trial % (n - 1)
            a = rng.uniform(-1, 1, size=(n, r)) @ rng.uniform(-1, 1, size=(r, n))
        u, s, vt = np.linalg.svd(a)
        tol = 1e-10 * s.max() * n
        want = vt.T @ np.diag([1 / x if x > tol else 0.0 for x in s]) @ u.T
        assert np.max(np.abs(oracle.pseudo_inverse(a) - want)) <= 1e-6


def test_partial_correlation_first_order(oracle):  # acceptance criterion 4a (acceptance_tests.cpp:222-240)
    rng = np.random.default_rng(40000)
    for idx in range(1000):
        n = 3 + idx % 5
        x = rng.normal(size=(n, 2 * n + 8))
        c = oracle.compute_correlation(x)
        i, j, k = idx % n, (idx % n + 1) % n, (idx % n + 2) % n
        want = (c[i, j] - c[i, k] * c[j, k]) / math.sqrt((1 - c[i, k] ** 2) * (1 - c[j, k] ** 2))
        got, deg = oracle.partial_correlation(c, i, j, [k])
        assert not deg and abs(got - want) <= 1e-10


def test_partial_correlation_residual_oracle(oracle):  # acceptance criterion 4b (acceptance_tests.cpp:242-262)
    for idx in range(100):
        seed = 50000 + idx
        w = oracle.random_dag(8, 0.3, seed)
        x = oracle.sample_linear_gaussian(w, 400, seed + 1)
        c = oracle.compute_correlation(x)
        base = idx % 4
        for ell in (2, 3):
            s = [base + 2 + k for k in range(ell)]
            xs = (x[s] - x[s].mean(axis=1, keepdims=True)).T
            xi = x[base] - x[base].mean()
            xj = x[base + 1] - x[base + 1].mean()
            ri = xi - xs @ np.linalg.lstsq(xs, xi, rcond=None)[0]
            rj = xj - xs @ np.linalg.lstsq(xs, xj, rcond=None)[0]
            want = ri @ rj / math.sqrt((ri @ ri) * (rj @ rj))
            got, _ = oracle.partial_correlation(c, base, base + 1, s)
            assert abs(got - want) <= 1e-6


def test_partial_correlation_symmetry_and_degenerate(oracle):  # test_stats.cpp:319-371
    rng = np.random.default_rng(7000)
    for _ in range(30):
        c = oracle.compute_correlation(rng.normal(size=(8, 24)))
        a, _ = oracle.partial_correlation(c, 0, 1, [2, 5, 7])
        b, _ = oracle.partial_correlation(c, 1, 0, [2, 5, 7])
        assert a == b
    c = make_correlation(3, [(0, 1, 0.5), (0, 2, 1.0), (1, 2, 0.5)])
    _, deg = oracle.partial_correlation(c, 0, 1, [2])
    assert deg
    ind, z, rho, deg = oracle.ci_test(c, 0, 1, [2], 10.0)
    assert not ind and deg and math.isinf(z)
    c = make_correlation(3, [(0, 1, 0.9)])
    ind, z, _, _ = oracle.ci_test(c, 0, 1, [], 0.062)
    assert not ind and abs(z - 1.4722194895832204) <= 1e-12
    ind, z, _, _ = oracle.ci_test(c, 0, 2, [], 0.062)
    assert ind and z == 0.0
    with pytest.raises(oracle.OracleError):
        oracle.ci_test(c, 1, 1, [2], 0.1)
    with pytest.raises(oracle.OracleError):
        oracle.ci_test(c, 0, 1, [0], 0.1)


# ------------------------------------------------------------------ datagen / rng
def test_datagen_determinism_and_shape(oracle):  # test_datagen.cpp
    a = oracle.random_dag(30, 0.3, 9)
    b = oracle.random_dag(30, 0.3, 9)
    assert np.array_equal(a, b) and not np.array_equal(a, oracle.random_dag(30, 0.3, 10))
    w = oracle.random_dag(40, 0.4, 123)
    assert not np.triu(w).any()
    nz = w[w != 0]
    assert nz.min() >= 0.1 and nz.max() < 1.0
    x1 = oracle.sample_linear_gaussian(oracle.random_dag(10, 0.3, 21), 200, 5)
    x2 = oracle.sample_linear_gaussian(oracle.random_dag(10, 0.3, 21), 200, 5)
    assert np.array_equal(x1, x2)
    cnt = (oracle.random_dag(1000, 0.1, 78) != 0).sum()
    assert abs(cnt - 49950) <= 4 * math.sqrt(49950 * 0.9)


# ------------------------------------------------------------------ skeleton
def test_star_graph(oracle):  # test_skeleton.cpp:102-127
    c = oracle.normalize_correlation(star_correlation())
    for strat in (oracle.SERIAL, oracle.EDGE, oracle.SET, oracle.KEYS):
        r = oracle.run_pc_stable(c, 1000, strategy=strat)
        assert r.edge_set() == [(0, 1), (0, 2), (0, 3)]
        assert r.levels_run() == 3 and r.stop_reason == "max-degree"
        assert [l.edges_removed for l in r.levels] == [1, 2, 0]
        assert r.sepsets == {(1, 2): (), (1, 3): (0,), (2, 3): (0,)}


def test_level_zero_counts(oracle):  # acceptance criterion 6
    for n in (10, 100, 500):
        r = oracle.run_pc_stable(np.eye(n), 100, alpha=0.05)
        assert r.levels[0].ci_tests == n * (n - 1) // 2
        assert r.adjacency.sum() == 0


def test_stop_conditions(oracle):  # test_skeleton.cpp:139-177
    c = oracle.normalize_correlation(star_correlation())
    r = oracle.run_pc_stable(c, 1000, max_level=1)
    assert r.levels_run() == 2 and r.stop_reason == "level-cap"
    c5 = make_correlation(5, [(i, j, 0.97) for i in range(5) for j in range(i + 1, 5)])
    r = oracle.run_pc_stable(c5, 5)
    assert r.stop_reason == "sample-size" and [l.edges_removed for l in r.levels] == [0, 10]
    with pytest.raises(oracle.OracleError):
        oracle.run_pc_stable(np.eye(3), 3)
    with pytest.raises(oracle.OracleError):
        oracle.run_pc_stable(np.eye(3), 100, alpha=2.0)


def test_chain_and_collider(oracle):  # acceptance criterion 8
    w = np.zeros((3, 3)); w[1, 0] = 0.8; w[2, 1] = 0.9
    r = oracle.run_pc_stable(oracle.compute_correlation(oracle.sample_linear_gaussian(w, 10000, 31)), 10000,
                             alpha=0.01)
    assert r.edge_set() == [(0, 1), (1, 2)] and r.sepsets[(0, 2)] == (1,)
    w = np.zeros((3, 3)); w[2, 0] = 0.8; w[2, 1] = 0.9
    r = oracle.run_pc_stable(oracle.compute_correlation(oracle.sample_linear_gaussian(w, 10000, 32)), 10000,
                             alpha=0.01)
    assert r.edge_set() == [(0, 2), (1, 2)] and r.sepsets[(0, 1)] == ()


def _audit(oracle, r, c, m, alpha):  # support.hpp:113-148 (criterion 7)
    p = c.shape[0]
    for i in range(p):
        for j in range(i + 1, p):
            s = r.sepsets.get((i, j))
            if r.adjacency[i, j]:
                assert s is None
                continue
            assert s is not None
            tau = oracle.threshold_tau(alpha, m, len(s))
            assert oracle.ci_test(c, i, j, list(s), tau)[0]


def test_strategy_equivalence_and_audit(oracle):  # acceptance criteria 1 and 7
    for inst in range(50):
        p = (20, 50, 100)[inst % 3]
        d = (0.1, 0.2, 0.3)[(inst // 3) % 3]
        c = instance(oracle, p, d, 1000, 1000 + inst)
        ref = oracle.run_pc_stable(c, 1000, alpha=0.05)
        if inst % 10 == 0:
            _audit(oracle, ref, c, 1000, 0.05)
        keys = oracle.run_pc_stable(c, 1000, alpha=0.05, strategy=oracle.KEYS, workers=4)
        assert keys.sepsets == ref.sepsets  # the serial rule, reproduced in parallel
        assert [(l.ci_tests, l.edges_removed) for l in keys.levels] == \
            [(l.ci_tests, l.edges_removed) for l in ref.levels]
        for strat in (oracle.EDGE, oracle.SET):
            for workers in (1, 4, 8):
                r = oracle.run_pc_stable(c, 1000, alpha=0.05, strategy=strat, workers=workers,
                                         schedule_seed=inst * 31 + workers)
                assert r.edge_set() == ref.edge_set()
                assert r.levels_run() == ref.levels_run() and r.stop_reason == ref.stop_reason


def test_tile_shape_invariance(oracle):  # test_skeleton.cpp:227-246
    c = instance(oracle, 15, 0.3, 800, 42)
    ref = oracle.run_pc_stable(c, 800, alpha=0.05)
    for beta in (1, 3, 100):
        assert oracle.run_pc_stable(c, 800, alpha=0.05, strategy=oracle.EDGE, workers=2,
                                    edges_per_unit=beta).edge_set() == ref.edge_set()
    for theta in (1, 7, 1000):
        for delta in (1, 2, 5):
            assert oracle.run_pc_stable(c, 800, alpha=0.05, strategy=oracle.SET, workers=2, unit_width=theta,
                                        set_groups=delta).edge_set() == ref.edge_set()


def test_level_keys_shards_compose(oracle):
    """Serial-rule keys of a level computed over edge shards equal the whole-level keys."""
    c = instance(oracle, 60, 0.2, 500, 5)
    r = oracle.run_pc_stable(c, 500, alpha=0.05, max_level=0)
    off = np.concatenate([[0], np.cumsum(r.adjacency.sum(axis=1))]).astype(np.int32)
    idx = np.concatenate([np.nonzero(r.adjacency[i])[0] for i in range(60)]).astype(np.int32)
    tau = oracle.threshold_tau(0.05, 500, 1)
    whole = oracle.level_keys(c, off, idx, 1, tau, threads=4)
    n = len(whole)
    parts = [oracle.level_keys(c, off, idx, 1, tau, e_begin=b, e_end=min(n, b + 97)) for b in range(0, n, 97)]
    assert np.array_equal(np.concatenate(parts), whole)
