"""How much the headline config's result depends on the correlation's summation order.

The reference leaves the Gram's order to Eigen (stats.hpp:137, untested bits); the device pins it
(FMA chain over k, restated by oracle compute_correlation_fma, tests/golden/*_full.npz).  This runs the
oracle's Strategy::Serial result (ORC_FAST) on the same data with the OTHER natural order -- sequential
two-rounding dot products (oracle compute_correlation, the reference's operation order without FMA) --
and reports, level by level, how many removed pairs / sepsets differ from the fixture.  Test
infrastructure; run in the CPU container:  python tools/corr_order_sensitivity.py C2 [--threads N]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402
from tests.golden_tools import canon_from_oracle  # noqa: E402
from tools.make_golden import ALPHA, CASES, case_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", default="C2", nargs="?")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    p, m, d, seed, max_level, _, _ = CASES[a.case]
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"{a.case.lower()}_full.npz")))
    x, _ = case_data(a.case)
    c_fma = O.compute_correlation_fma(x, threads=a.threads)
    c_seq = O.compute_correlation(x, threads=a.threads)
    diff = c_fma != c_seq
    t0 = time.time()
    r = O.run_pc_stable_arrays(c_seq, m, alpha=ALPHA, max_level=max_level, strategy=O.FAST, workers=a.threads)
    can = canon_from_oracle(r)
    out = {"case": a.case, "corr_entries_differing": int(diff.sum()), "corr_entries": int(p * p),
           "max_abs_corr_diff": float(np.abs(c_fma - c_seq).max()), "oracle_seconds": time.time() - t0,
           "levels": []}
    for ell in [int(v) for v in g["levels"]]:
        gk = g.get(f"keys_{ell}")
        dk, dm = can.blocks.get(ell, (np.zeros(0, np.int64), np.zeros((0, ell), np.int32)))
        ent = {"level": ell, "removed_seq_order": int(len(dk))}
        cnt = [row for row in g["counters"] if int(row[0]) == ell]
        if cnt:
            ent["removed_fma_order"] = int(cnt[0][3])
            ent["ci_tests_fma_order"] = int(cnt[0][1])
        lv = [l for l in r.levels if l.level == ell]
        if lv:
            ent["ci_tests_seq_order"] = int(lv[0].ci_tests)
        if gk is not None:
            gm = g[f"members_{ell}"].astype(np.int32)
            common, gi, di = np.intersect1d(gk, dk, return_indices=True)
            ent["pairs_removed_only_in_fma_order"] = int(len(gk) - len(common))
            ent["pairs_removed_only_in_seq_order"] = int(len(dk) - len(common))
            ent["same_pair_different_sepset"] = int((gm[gi] != dm[di]).any(axis=1).sum()) if ell else 0
        out["levels"].append(ent)
    out["edges_left_fma_order"] = int(g["edges_left"])
    out["edges_left_seq_order"] = int(len(can.edges))
    out["rows_differing"] = int((can.row_hash() != g["row_hash"]).sum())
    print(json.dumps(out, indent=1))
    json.dump(out, open(os.path.join(ROOT, "profiles", f"r2_{a.case.lower()}_corr_order_sensitivity.json"), "w"),
              indent=1)


if __name__ == "__main__":
    main()
