"""Disjoint instances on concurrent host threads (the reference is documented as safe for that,
SPEC.md:394): two threads each run whole skeletons through the library at the same time -- separate
sessions, streams, counters and pinned slots -- and every result equals the same run done alone."""
import threading

import numpy as np
import pytest

from tests.helpers import instance

pytestmark = pytest.mark.gpu


def _run(pcs, c, m, variant):
    r = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=0.01, strategy=pcs.Strategy(variant)))
    return r.skeleton.cells.copy(), r.sepsets.as_dict(), [(l.level, l.ci_tests, l.edges_removed) for l in r.levels]


def test_concurrent_sessions_match_sequential(pcs, oracle):
    cases = [(instance(oracle, 150, 0.1, 600, 31), 600, "set"), (instance(oracle, 220, 0.05, 400, 32), 400, "edge"),
             (instance(oracle, 120, 0.2, 300, 33), 300, "set"), (instance(oracle, 90, 0.3, 800, 34), 800, "edge")]
    alone = [_run(pcs, c, m, v) for c, m, v in cases]
    out = [None] * (2 * len(cases))
    errs = []

    def worker(k):
        try:
            for rep in range(2):
                c, m, v = cases[(k + rep) % len(cases)]
                out[2 * k + rep] = ((k + rep) % len(cases), _run(pcs, c, m, v))
        except Exception as e:  # surfaced below
            errs.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(cases))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errs, errs
    for idx, (cells, sep, levels) in out:
        a_cells, a_sep, a_levels = alone[idx]
        assert np.array_equal(cells, a_cells) and sep == a_sep and levels == a_levels, f"case {idx}"
