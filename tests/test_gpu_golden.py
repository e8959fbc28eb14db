"""Whole-run parity against committed golden fixtures (tests/golden/*_full.npz, made by
tools/make_golden.py from the CPU oracle) -- the bench's own pipeline, end to end.

Each case runs the device exactly as bench.py does: data -> device correlation (FMA-chain Gram,
corr.cu) -> run_pc_stable, and compares the WHOLE result with the oracle's Strategy::Serial result
on the same data: every level's removed pairs and serial-rule sepsets, per-level ci_tests /
pseudo_inverses / edges_removed, the remaining edges and the stop reason (tests/golden_tools.py).
The device correlation matrix is first checked bit for bit against the oracle's restatement of the
device order (pyoracle.compute_correlation_fma), so the fixtures' correlation and the device's are
the same bits.  C2 is BASELINE configs[1] (the bench headline, capped at level 3 like the bench);
C5_2000 / C5_5000 / C5_10000 are scaling-sweep shapes (levels 0-2 / 0-1 / 0-1; the last runs the tiled
level-1 kernel over 157 target bands, i.e. ten L2 groups)."""
import hashlib
import os
import time

import numpy as np
import pytest

from tests.golden_tools import canon_from_device, compare

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
THREADS = max(1, min(16, os.cpu_count() or 1))


def _load(name):
    path = os.path.join(GOLD, f"{name.lower()}_full.npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {path} not generated")
    return dict(np.load(path))


def _data(pcs, oracle, g):
    p, m, d, seed = int(g["p"]), int(g["m"]), float(g["density"]), int(g["seed"])
    if bool(g["rescaled"]) and p >= 10000:  # the device generator (bit-identical, test_gpu_datagen.py)
        import torch

        w = pcs.random_dag(p, d, seed)
        xd = torch.empty((p, m), dtype=torch.float64, device="cuda")
        pcs.sample_linear_gaussian_device(w, m, seed + 1, xd.data_ptr(), rescaled=True)
        x = xd.cpu().numpy()
    elif bool(g["rescaled"]):
        w = pcs.random_dag(p, d, seed)
        x, _ = pcs.sample_linear_gaussian_rescaled(w, m, seed + 1)
        x = np.ascontiguousarray(np.asarray(x).T)
    else:
        w = oracle.random_dag(p, d, seed)
        x = oracle.sample_linear_gaussian(w, m, seed + 1)
    assert hashlib.sha256(x.tobytes()).hexdigest() == str(g["data_sha256"]), "generator output changed"
    return x  # (p, m): row j = variable j


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5_2000"])
def test_device_correlation_bits(pcs, oracle, name):
    g = _load(name)
    x = _data(pcs, oracle, g)
    dev = pcs.compute_correlation(x.T)
    ref = oracle.compute_correlation_fma(x, threads=THREADS)
    bad = int((dev.view(np.int64) != ref.view(np.int64)).sum())
    assert bad == 0, f"{name}: {bad} correlation entries differ from the oracle's FMA-order restatement"
    assert hashlib.sha256(dev.tobytes()).hexdigest() == str(g["corr_sha256"])


@pytest.mark.parametrize("name,variant", [("C1", "set"), ("C1", "edge"), ("C3", "set"), ("C3", "edge"),
                                          ("C4", "set"), ("C4", "edge"), ("C2", "set"), ("C5_2000", "set"),
                                          ("C5_5000", "set"), ("C5_10000", "set")])
def test_whole_run_matches_golden(pcs, oracle, name, variant):
    g = _load(name)
    x = _data(pcs, oracle, g)
    ml = int(g["max_level"])
    cfg = pcs.SkeletonConfig(alpha=float(g["alpha"]), max_level=None if ml < 0 else ml,
                             strategy=pcs.Strategy(variant))
    t0 = time.time()
    res = pcs.run_pc_stable_data(x.T, cfg)
    dt = time.time() - t0
    errs = compare(canon_from_device(res), g)
    assert not errs, f"{name} {variant}: " + "; ".join(errs)
    print(f"{name} {variant}: whole run identical to the oracle ({res.levels_run()} levels, "
          f"{sum(l.ci_tests for l in res.levels):.3e} serial CI tests, {res.skeleton.edge_count()} edges) "
          f"in {dt:.2f}s")
