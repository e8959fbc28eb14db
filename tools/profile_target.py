"""ncu target: BASELINE C2 levels 0..L-1 in full, then level L pass 0 on 1/S of the work units
(so one launch of the dominant kernel is short enough for --set full replays).
usage: python tools/profile_target.py [level=3] [slices=32] [variant=set]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_08491_b200 as pcs

level = int(sys.argv[1]) if len(sys.argv) > 1 else 3
slices = int(sys.argv[2]) if len(sys.argv) > 2 else 32
variant = sys.argv[3] if len(sys.argv) > 3 else "set"
p, m, d, seed = 1000, 10000, 0.1, 7919
w = pcs.random_dag(p, d, seed)
x = pcs.sample_linear_gaussian(w, m, seed + 1)
c = pcs.compute_correlation(x)
s = pcs.Session(c, m, pcs.SkeletonConfig(alpha=0.01, strategy=pcs.Strategy(variant)))
while True:
    run, ell, nk = s.level_begin()
    if ell == level:
        s.set_shard(0, slices)
        s.level_pass(0)
        s.keys()
        s.level_end()
        l = s.finish(with_sepsets=False).levels[-1]
        print("profiled level", ell, "keys", nk, "device tests", l.device_ci_tests, "exact", l.device_exact_tests,
              "pinv", l.device_pseudo_inverses, "kernel_ms", l.kernel_ms)
        break
    s.level_pass(0); s.level_pass(1); s.level_end()
