"""Orientation (orient.hpp) on the device path vs the oracle restatement.

Bar: the MixedGraph (directed and undirected pair sets) identical to the oracle's on the same
skeleton and sepsets -- the reference's own orientation tests (test_orient.cpp), skeletons of
seeded instances computed by the device, random sepsets that produce conflicting votes, and
random partially directed graphs for apply_meek_rules alone."""
import numpy as np
import pytest

from tests.helpers import instance

pytestmark = pytest.mark.gpu


def skel(n, edges):
    a = np.zeros((n, n), np.uint8)
    for i, j in edges:
        a[i, j] = a[j, i] = 1
    return a


def same(dev, ref):
    assert sorted(dev.directed) == ref.directed, (sorted(dev.directed), ref.directed)
    assert sorted(dev.undirected) == ref.undirected, (sorted(dev.undirected), ref.undirected)


def test_reference_orientation_cases(pcs, oracle):
    """test_orient.cpp:25-181 through the product API."""
    M = pcs.MixedGraph
    assert pcs.find_v_structures(skel(3, [(0, 2), (1, 2)]), {(0, 1): ()}) == M(3, [(0, 2), (1, 2)])
    assert pcs.find_v_structures(skel(3, [(0, 2), (1, 2)]), {(0, 1): (2,)}) == M(3, [], [(0, 2), (1, 2)])
    g = pcs.find_v_structures(skel(3, [(0, 1), (0, 2), (1, 2)]), {})
    assert not g.directed and len(g.undirected) == 3
    g = pcs.find_v_structures(skel(4, [(0, 1), (1, 2), (0, 3)]), {(0, 2): (), (1, 3): ()})
    assert g.has_undirected(0, 1) and g.has_directed(2, 1) and g.has_directed(3, 0)
    with pytest.raises(ValueError):
        pcs.find_v_structures(skel(3, [(0, 2), (1, 2)]), {})
    assert pcs.apply_meek_rules(M(3, [(0, 1)], [(1, 2)])) == M(3, [(0, 1), (1, 2)])
    g = M(3, [(0, 1)], [(1, 2), (0, 2)])
    assert pcs.apply_meek_rules(g) == g
    assert pcs.apply_meek_rules(M(3, [(0, 1), (1, 2)], [(0, 2)])) == M(3, [(0, 1), (1, 2), (0, 2)])
    assert pcs.apply_meek_rules(M(4, [(2, 1), (3, 1)], [(0, 1), (0, 2), (0, 3)])) == \
        M(4, [(0, 1), (2, 1), (3, 1)], [(0, 2), (0, 3)])
    assert pcs.apply_meek_rules(M(4, [(2, 3), (3, 1)], [(0, 1), (0, 2)])) == M(4, [(0, 1), (2, 3), (3, 1)], [(0, 2)])
    g = M(4, [], [(0, 1), (1, 2), (2, 3)])
    assert pcs.apply_meek_rules(g) == g
    assert pcs.orient_skeleton(skel(4, [(0, 1), (1, 2), (2, 3)]), {(0, 2): (), (1, 3): (2,)}) == \
        M(4, [(0, 1), (2, 1)], [(2, 3)])
    once = pcs.apply_meek_rules(M(4, [(2, 1), (3, 1)], [(0, 1), (0, 2), (0, 3)]))
    assert pcs.apply_meek_rules(once) == once


@pytest.mark.parametrize("p,d,m,seed", [(12, 0.25, 800, 5), (100, 2.0 / 99.0, 1000, 0), (50, 0.2, 1000, 1003),
                                        (100, 0.3, 1000, 1008), (60, 0.4, 500, 78)])
def test_orient_device_result_matches_oracle(pcs, oracle, p, d, m, seed):
    """Device skeleton + sepsets (record form, level-0 removals implied) -> orient_skeleton."""
    c = instance(oracle, p, d, m, seed)
    r = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=0.05))
    dev = pcs.orient_skeleton(r.skeleton, r.sepsets)
    ref = oracle.orient(p, r.skeleton.cells, r.sepsets.as_dict(), stage=3)
    same(dev, ref)
    v = pcs.find_v_structures(r.skeleton, r.sepsets)
    same(v, oracle.orient(p, r.skeleton.cells, r.sepsets.as_dict(), stage=1))


def test_orient_random_sepsets_conflicts(pcs, oracle):
    """Random skeletons with random sepsets: many conflicting votes, rules 1-4 all firing."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(5, 40))
        a = np.triu(rng.random((n, n)) < rng.uniform(0.05, 0.5), 1)
        a = (a | a.T).astype(np.uint8)
        sep = {}
        for i in range(n):
            for j in range(i + 1, n):
                if not a[i, j]:
                    k = int(rng.integers(0, 4))
                    sep[(i, j)] = tuple(sorted(rng.choice([v for v in range(n) if v not in (i, j)],
                                                          size=min(k, n - 2), replace=False).tolist()))
        ref = oracle.orient(n, a, sep, stage=3)
        same(pcs.orient_skeleton(a, sep), ref)


def test_meek_random_partial_orientations(pcs, oracle):
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(4, 30))
        a = np.triu(rng.random((n, n)) < rng.uniform(0.1, 0.5), 1)
        edges = [(i, j) for i in range(n) for j in range(i + 1, n) if a[i, j]]
        perm = rng.permutation(n)  # orient along a random order -> acyclic partial orientation
        directed = [((i, j) if perm[i] < perm[j] else (j, i)) for i, j in edges if rng.random() < 0.3]
        undirected = [e for e in edges if (e not in directed and (e[1], e[0]) not in directed)]
        g = pcs.MixedGraph(n, directed, undirected)
        ref = oracle.orient(n, (a | a.T).astype(np.uint8), {}, stage=2, directed=sorted(directed))
        same(pcs.apply_meek_rules(g), ref)


def test_orient_c3_shape(pcs, oracle):
    """DREAM5 shape (p = 1643, m = 850, d = 0.01): the bench workload's own skeleton."""
    p, m = 1643, 850
    w = pcs.random_dag(p, 0.01, 7919 * 2)
    x = pcs.sample_linear_gaussian(w, m, 7919 * 2 + 1)
    r = pcs.run_pc_stable_data(x, pcs.SkeletonConfig(alpha=0.01))
    dev = pcs.orient_skeleton(r.skeleton, r.sepsets)
    ref = oracle.orient(p, r.skeleton.cells, r.sepsets.as_dict(), stage=3)
    same(dev, ref)
    assert len(dev.directed) + len(dev.undirected) == r.skeleton.edge_count()
