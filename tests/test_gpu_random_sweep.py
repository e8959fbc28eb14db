"""Randomised whole-run parity: seeded random shapes (p 20-400, density 0.02-0.5, m 20-2000, alpha
0.01-0.1, some level caps), device vs the oracle's Strategy::Serial result (ORC_FAST) on the same
correlation bits -- skeleton, every level's sepsets, per-level counters, stop reason.  Dense small-m
shapes reach deep levels (the generic-ell kernel beyond l = 8); a subprocess repeats a subset with the
tiled level-1 kernel forced on (PCS_L1_TILE=1), since its p >= 2048 rule keeps it off these sizes."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.golden_tools import canon_from_device, canon_from_oracle, compare, summary
from tests.helpers import instance

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        d = float(rng.choice([0.02, 0.05, 0.1, 0.2, 0.35, 0.5]))
        dense = d >= 0.2
        p = int(rng.integers(20, 80 if dense else 400))
        m = int(rng.choice([30, 80, 200, 800, 2000]))
        alpha = float(rng.choice([0.01, 0.05, 0.1]))
        # dense rows keep C(w, l) sets per row large for many levels: cap them (the oracle's time)
        cap = int(rng.integers(2, 6)) if dense else (None if rng.random() < 0.7 else int(rng.integers(1, 4)))
        out.append((p, d, m, alpha, cap, 1000 + k))
    return out


def _check(pcs, oracle, p, d, m, alpha, cap, seed, variant):
    c = instance(oracle, p, d, m, seed)
    ref = oracle.run_pc_stable_arrays(c, m, alpha=alpha, max_level=cap, strategy=oracle.FAST, workers=4)
    dev = pcs.run_pc_stable(c, m, pcs.SkeletonConfig(alpha=alpha, max_level=cap, strategy=pcs.Strategy(variant)))
    return compare(canon_from_device(dev), summary(canon_from_oracle(ref))), len(ref.levels)


@pytest.mark.parametrize("variant", ["set", "edge"])
def test_random_shapes(pcs, oracle, variant):
    deepest = 0
    for case in _cases(24, 7 if variant == "set" else 8):
        errs, nlev = _check(pcs, oracle, *case, variant)
        assert not errs, f"{case} {variant}: {errs}"
        deepest = max(deepest, nlev - 1)
    print(f"{variant}: 24 random shapes identical, deepest level {deepest}")


def _sweep_subprocess(env_extra, variant, n, seed):
    code = (
        "import sys, json; sys.path.insert(0, %r)\n"
        "import paper_1812_08491_b200 as pcs\n"
        "from oracle import pyoracle as O\n"
        "from tests.test_gpu_random_sweep import _cases, _check\n"
        "bad = []\n"
        "for case in _cases(%d, %d):\n"
        "    errs, _ = _check(pcs, O, *case, %r)\n"
        "    if errs: bad.append([list(case), errs])\n"
        "print(json.dumps(bad))\n" % (ROOT, n, seed, variant))
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_random_shapes_unstaged_edge():
    """cuPC-E on the unstaged level_edge_kernel (the fallback for rows too wide for shared memory)."""
    assert _sweep_subprocess({"PCS_EDGE_STAGED": "0"}, "edge", 10, 11) == []


def test_random_shapes_tiled_level1():
    code = (
        "import sys, json; sys.path.insert(0, %r)\n"
        "import paper_1812_08491_b200 as pcs\n"
        "from oracle import pyoracle as O\n"
        "from tests.test_gpu_random_sweep import _cases, _check\n"
        "bad = []\n"
        "for case in _cases(10, 9):\n"
        "    errs, _ = _check(pcs, O, *case, 'set')\n"
        "    if errs: bad.append([list(case), errs])\n"
        "print(json.dumps(bad))\n" % ROOT)
    env = dict(os.environ, PCS_L1_TILE="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=ROOT, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    bad = json.loads(out.stdout.strip().splitlines()[-1])
    assert bad == [], bad
