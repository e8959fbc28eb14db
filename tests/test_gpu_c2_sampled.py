"""Parity at BASELINE config C2's full size (p=1000, m=10000, d=0.1, alpha=0.01, bench seed 7919).

C2 sits in the reference's rank-truncation regime (a third of all pairs at the rho
clamp, pseudo-inverses dropping columns, degenerate H everywhere), so it is the hardest input for
bit parity.  The whole skeleton is out of the oracle's reach (level 3 alone is 7.9e11 serial CI
tests), so this test checks:
  * levels 0-1 in full: skeleton, sepsets and counters identical to the oracle's serial rule;
  * levels 2 and 3 on samples of the device's own snapshot: the device's per-edge keys (serial-rule
    first separating set, both directions) identical to the oracle's `level_keys` for the same
    edges, which exercises the cuPC-S kernel's certified filter and its exact fallback.
Both sides consume the same correlation matrix bits (the oracle's)."""
import time

import numpy as np
import pytest

from tests.helpers import assert_same_result, instance

pytestmark = pytest.mark.gpu

P, M, D, SEED, ALPHA = 1000, 10000, 0.1, 7919, 0.01


@pytest.fixture(scope="module")
def c2(oracle):
    return instance(oracle, P, D, M, SEED)


def _device_keys(ptr: int, n: int) -> np.ndarray:
    import torch

    from paper_1812_08491_b200.multigpu import _CudaArray

    return torch.as_tensor(_CudaArray(ptr, n), device="cuda").cpu().numpy().copy()


NONE = (1 << 63) - 1


def _full_row_keys(oracle, ref, e0, a, b, off, idx, ell):
    """The oracle's keys carry the reduced rank (test_edge_over_sets' rank among the sets of row r
    minus the target, skeleton.hpp:140-149); the device keys carry the rank among all ell-subsets of
    row r (order-isomorphic).  Convert oracle -> full-row rank."""
    from math import comb

    out = ref.copy()
    for k in np.nonzero(ref != NONE)[0]:
        key = int(ref[k])
        d, rk = key >> 62, key & ((1 << 62) - 1)
        r, other = (a[e0 + k], b[e0 + k]) if d == 0 else (b[e0 + k], a[e0 + k])
        row = idx[off[r]:off[r + 1]]
        w = len(row)
        q = int(np.searchsorted(row, other))
        pos = oracle.unrank_positions_excluding(w - 1, ell, rk, q)
        full = comb(w, ell) - 1 - sum(comb(w - 1 - int(pos[t]), ell - t) for t in range(ell))
        out[k] = (d << 62) | full
    return out


def test_c2_levels_0_1_full(pcs, oracle, c2):
    ref = oracle.run_pc_stable(c2, M, alpha=ALPHA, max_level=1, strategy=oracle.KEYS, workers=8)
    dev = pcs.run_pc_stable(c2, M, pcs.SkeletonConfig(alpha=ALPHA, max_level=1))
    assert_same_result(dev, ref, label="C2 levels 0-1")


@pytest.mark.parametrize("variant,top", [("set", 3), ("edge", 2)])
def test_c2_levels_2_3_sampled_keys(pcs, oracle, c2, variant, top):
    """cuPC-S through level 3; cuPC-E (a pseudo-inverse per test) through level 2."""
    from math import comb

    s = pcs.Session(c2, M, pcs.SkeletonConfig(alpha=ALPHA, max_level=top, strategy=pcs.Strategy(variant)))
    checked = {}
    try:
        while True:
            running, ell, nkeys = s.level_begin()
            if not running:
                break
            for ps in (0, 1):
                s.level_pass(ps)
            if ell >= 2:
                off, idx = s.snapshot(P)
                ptr, n = s.keys()
                keys = _device_keys(ptr, n)
                tau = oracle.threshold_tau(ALPHA, M, ell)
                # per-edge oracle cost (both directions, no early exit) -> pick cheap-to-moderate edges
                rows = np.repeat(np.arange(P), np.diff(off))
                a = rows[idx > rows]
                b = idx[idx > rows]
                wd = np.diff(off)
                cost = np.array([comb(int(wd[x]) - 1, ell) + comb(int(wd[y]) - 1, ell) for x, y in zip(a, b)],
                                dtype=float)
                budget = 4e8 if ell == 3 else 2e8  # oracle serial tests (~10 s on 8 threads)
                starts = np.linspace(0, n - 1, 24).astype(int)
                per_range = budget / len(starts)
                nchk, nrem = 0, 0
                t0 = time.time()
                for st in starts:
                    lim = min(n, st + 256)
                    while st < lim and cost[st] > per_range:  # skip edges too costly for the oracle
                        st += 1
                    e1, spent = st, 0.0
                    while e1 < lim and e1 < st + 64 and spent + cost[e1] <= per_range:
                        spent += cost[e1]
                        e1 += 1
                    if e1 == st:
                        continue
                    ref = oracle.level_keys(c2, off, idx, ell, tau, int(st), int(e1), threads=8)
                    ref = _full_row_keys(oracle, ref, int(st), a, b, off, idx, ell)
                    got = keys[st:e1]
                    bad = np.nonzero(ref != got)[0]
                    assert len(bad) == 0, (f"level {ell} edges {st + bad[:5]}: device {got[bad[:5]]} "
                                           f"oracle {ref[bad[:5]]}")
                    nchk += e1 - st
                    nrem += int((ref != NONE).sum())
                checked[ell] = (nchk, nrem, time.time() - t0)
            s.level_end()
    finally:
        s.close()
    assert set(checked) == set(range(2, top + 1)), checked
    assert all(v[0] >= 50 for v in checked.values()), checked
    print(f"C2 {variant}: checked edges per level {checked}")
