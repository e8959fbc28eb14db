"""Dump the device correlation matrix (pcs.compute_correlation) for BASELINE configs so the oracle's
order can be checked against the device bits offline.  Writes gpurun_out/corr_<cfg>.npy."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08491_b200 as pcs  # noqa: E402

CFGS = {"C1": (100, 2 / 99, 1000, 0), "C2": (1000, 0.1, 10000, 7919), "C3": (1643, 0.01, 850, 7919 * 2),
        "C4": (5361, 0.002, 63, 7919 * 3)}
os.makedirs("gpurun_out", exist_ok=True)
for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else CFGS):
    p, d, m, seed = CFGS[name]
    w = pcs.random_dag(p, d, seed)
    x = pcs.sample_linear_gaussian(w, m, seed + 1)
    c = pcs.compute_correlation(x)
    np.save(f"gpurun_out/corr_{name}.npy", c)
    print(name, c.shape, float(np.abs(c - c.T).max()))
