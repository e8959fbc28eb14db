"""Orientation oracle (oracle/pcs_orient_oracle.c) pinned to the reference's own tests
(/root/reference/proj/tests/test_orient.cpp); CPU only."""
import numpy as np
import pytest

from tests.helpers import instance


def skel(n, edges):
    a = np.zeros((n, n), np.uint8)
    for i, j in edges:
        a[i, j] = a[j, i] = 1
    return a


def test_empty_separating_set_makes_a_collider(oracle):  # test_orient.cpp:25-34
    g = oracle.orient(3, skel(3, [(0, 2), (1, 2)]), {(0, 1): ()}, stage=1)
    assert g == oracle.MixedGraph(3, [(0, 2), (1, 2)], [])


def test_middle_vertex_in_separating_set_blocks_the_collider(oracle):  # :36-46
    g = oracle.orient(3, skel(3, [(0, 2), (1, 2)]), {(0, 1): (2,)}, stage=1)
    assert g == oracle.MixedGraph(3, [], [(0, 2), (1, 2)])


def test_shielded_triple_is_never_oriented(oracle):  # :48-56
    g = oracle.orient(3, skel(3, [(0, 1), (0, 2), (1, 2)]), {}, stage=1)
    assert g.directed == [] and len(g.undirected) == 3


def test_conflicting_votes_leave_the_edge_undirected(oracle):  # :58-71
    g = oracle.orient(4, skel(4, [(0, 1), (1, 2), (0, 3)]), {(0, 2): (), (1, 3): ()}, stage=1)
    assert (0, 1) in g.undirected and (2, 1) in g.directed and (3, 0) in g.directed


def test_missing_separating_set_is_an_error(oracle):  # :73-79
    with pytest.raises(oracle.OracleError):
        oracle.orient(3, skel(3, [(0, 2), (1, 2)]), {}, stage=1)


@pytest.mark.parametrize("case", ["r1", "r1_shield", "r2", "r3", "r4", "none", "tail", "idem"])
def test_meek_rules(oracle, case):  # :81-181
    if case == "r1":
        g = oracle.orient(3, skel(3, [(0, 1), (1, 2)]), {}, stage=2, directed=[(0, 1)])
        assert g == oracle.MixedGraph(3, [(0, 1), (1, 2)], [])
    elif case == "r1_shield":
        g = oracle.orient(3, skel(3, [(0, 1), (1, 2), (0, 2)]), {}, stage=2, directed=[(0, 1)])
        assert g == oracle.MixedGraph(3, [(0, 1)], [(1, 2), (0, 2)])
    elif case == "r2":
        g = oracle.orient(3, skel(3, [(0, 1), (1, 2), (0, 2)]), {}, stage=2, directed=[(0, 1), (1, 2)])
        assert g == oracle.MixedGraph(3, [(0, 1), (1, 2), (0, 2)], [])
    elif case == "r3":
        g = oracle.orient(4, skel(4, [(2, 1), (3, 1), (0, 1), (0, 2), (0, 3)]), {}, stage=2, directed=[(2, 1), (3, 1)])
        assert g == oracle.MixedGraph(4, [(0, 1), (2, 1), (3, 1)], [(0, 2), (0, 3)])
    elif case == "r4":
        g = oracle.orient(4, skel(4, [(2, 3), (3, 1), (0, 1), (0, 2)]), {}, stage=2, directed=[(2, 3), (3, 1)])
        assert g == oracle.MixedGraph(4, [(0, 1), (2, 3), (3, 1)], [(0, 2)])
    elif case == "none":
        g = oracle.orient(4, skel(4, [(0, 1), (1, 2), (2, 3)]), {}, stage=2)
        assert g == oracle.MixedGraph(4, [], [(0, 1), (1, 2), (2, 3)])
    elif case == "tail":
        g = oracle.orient(4, skel(4, [(0, 1), (1, 2), (2, 3)]), {(0, 2): (), (1, 3): (2,)}, stage=3)
        assert g == oracle.MixedGraph(4, [(0, 1), (2, 1)], [(2, 3)])
    else:
        s = skel(4, [(2, 1), (3, 1), (0, 1), (0, 2), (0, 3)])
        once = oracle.orient(4, s, {}, stage=2, directed=[(2, 1), (3, 1)])
        twice = oracle.orient(4, s, {}, stage=2, directed=once.directed)
        assert once == twice


def test_preserves_the_skeleton_exactly(oracle):  # :183-202 (random_dag(12, .25, 5), m = 800)
    c = instance(oracle, 12, 0.25, 800, 5)
    r = oracle.run_pc_stable(c, 800)
    g = oracle.orient(12, r.adjacency, r.sepsets, stage=3)
    assert len(g.directed) + len(g.undirected) == int(np.triu(r.adjacency, 1).sum())
    adj = {(a, b) for a, b in g.directed} | {(b, a) for a, b in g.directed}
    adj |= {(a, b) for a, b in g.undirected} | {(b, a) for a, b in g.undirected}
    for i in range(12):
        for j in range(i + 1, 12):
            assert ((i, j) in adj) == bool(r.adjacency[i, j])
    for a, b in g.directed:
        assert (b, a) not in g.directed and (min(a, b), max(a, b)) not in g.undirected
