"""Generates tests/golden/c2_level3_snapshot.npz: the CSR snapshot (compact(), core.hpp:227-239)
at the start of level 3 of BASELINE config C2 (p=1000, m=10000, d=0.1, alpha=0.01, seed 7919),
produced by the device path.  bench.py's CPU baseline times the reference's level 3 on rows of
this snapshot (a bounded sample of the workload).  Requires a GPU."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_1812_08491_b200 as pcs

p, m, d, seed, level = 1000, 10000, 0.1, 7919, 3
w = pcs.random_dag(p, d, seed)
x = pcs.sample_linear_gaussian(w, m, seed + 1)
c = pcs.compute_correlation(x)
s = pcs.Session(c, m, pcs.SkeletonConfig(alpha=0.01))
while True:
    run, ell, nk = s.level_begin()
    assert run
    if ell == level:
        off, idx = s.snapshot(p)
        break
    s.level_pass(0); s.level_pass(1); s.level_end()
out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c2_level3_snapshot.npz")
np.savez_compressed(out, offsets=off, indices=idx, level=level, p=p, m=m, density=d, seed=seed)
print(out, off[-1], np.diff(off).max())
