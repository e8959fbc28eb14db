"""Generate whole-run golden fixtures from the CPU oracle (run HERE, in the CPU container; the
fixtures are committed under tests/golden/ and the GPU tests compare the device against them).

Each case: data from the reference generator (random_dag + sample_linear_gaussian, or the
overflow-safe rescaled variant for the C5 sweep shapes), correlation in the device's pinned order
(oracle compute_correlation_fma: tree means + FMA-chain Gram -- bit-identical to the device's C),
then the oracle's run_pc_stable with Strategy::Serial semantics (set-shared key mode ORC_FAST,
result-identical to Serial) up to the case's level cap.  Stored: per-level counters, stop reason,
per-level SHA-256 of (removed pairs, sepsets), remaining-edge digest, per-row hashes, and for the
listed levels the full removed-pair / sepset arrays (tests/golden_tools.py).

usage: python tools/make_golden.py C2 [C5_2000 ...] [--threads N]
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402
from tests.golden_tools import canon_from_oracle, summary  # noqa: E402

# name: (p, m, density, seed, max_level, rescaled generator, levels stored in full)
CASES = {
    "C1": (100, 1000, 2.0 / 99.0, 0, None, False, (1, 2, 3, 4)),
    "C2": (1000, 10000, 0.1, 7919, 3, False, (2, 3)),
    "C3": (1643, 850, 0.01, 2 * 7919, None, False, (2, 3, 4, 5, 6, 7, 8, 9)),
    "C4": (5361, 63, 0.002, 3 * 7919, None, False, (2, 3, 4)),
    "C5_2000": (2000, 5000, 0.05, 4 * 7919, 2, True, ()),
    "C5_5000": (5000, 5000, 0.05, 4 * 7919, 1, True, ()),
    "C5_10000": (10000, 5000, 0.05, 7 * 7919, 1, True, ()),
}
ALPHA = 0.01


def case_data(name):
    """(p, m) data of a case as variable-major (p, m) float64, plus the data's SHA-256."""
    p, m, d, seed, _, rescaled, _ = CASES[name]
    if rescaled:
        import paper_1812_08491_b200 as pcs  # host-side generator only (datagen.cpp); no device use
        w = pcs.random_dag(p, d, seed)
        x, _ = pcs.sample_linear_gaussian_rescaled(w, m, seed + 1)
        x = np.ascontiguousarray(np.asarray(x).T)
    else:
        w = O.random_dag(p, d, seed)
        x = O.sample_linear_gaussian(w, m, seed + 1)
    return x, hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def snapshots(name, threads, levels=(1, 2, 3)):
    """The live graph at the start of each listed level (compact()'s input, core.hpp:227-239), as
    packed upper-triangle bits -- the per-level work bench.py's reference arm samples rows from."""
    p, m, d, seed, _, _, _ = CASES[name]
    x, xsha = case_data(name)
    c = O.compute_correlation_fma(x, threads=threads)
    iu, ju = np.triu_indices(p, 1)
    out = {"p": np.int64(p), "levels": np.asarray(levels, np.int64), "data_sha256": np.array(xsha)}
    for ell in levels:
        r = O.run_pc_stable_arrays(c, m, alpha=ALPHA, max_level=ell - 1, strategy=O.FAST, workers=threads)
        out[f"adj_{ell}"] = np.packbits(r.adjacency[iu, ju])
        print(f"{name} snapshot at level {ell}: {int(r.adjacency[iu, ju].sum())} edges", flush=True)
    path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_snapshots.npz")
    np.savez_compressed(path, **out)
    print(f"-> {os.path.relpath(path, ROOT)} ({os.path.getsize(path) / 1e6:.2f} MB)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--snapshots", action="store_true", help="write <case>_snapshots.npz instead")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    if a.snapshots:
        for name in a.cases:
            snapshots(name, a.threads)
        return
    for name in a.cases:
        p, m, d, seed, max_level, rescaled, full = CASES[name]
        t0 = time.time()
        x, xsha = case_data(name)
        c = O.compute_correlation_fma(x, threads=a.threads)
        csha = hashlib.sha256(c.tobytes()).hexdigest()
        del x
        t1 = time.time()
        r = O.run_pc_stable_arrays(c, m, alpha=ALPHA, max_level=max_level, strategy=O.FAST, workers=a.threads)
        t2 = time.time()
        can = canon_from_oracle(r)
        out = summary(can, full)
        out.update(dict(m=np.int64(m), density=np.float64(d), seed=np.int64(seed), alpha=np.float64(ALPHA),
                        max_level=np.int64(-1 if max_level is None else max_level), rescaled=np.bool_(rescaled),
                        data_sha256=np.array(xsha), corr_sha256=np.array(csha),
                        oracle_seconds=np.float64(t2 - t1), threads=np.int64(a.threads)))
        path = os.path.join(ROOT, "tests", "golden", f"{name.lower()}_full.npz")
        np.savez_compressed(path, **out)
        lv = ", ".join(f"L{l.level}: {l.ci_tests:.3e} tests, {l.edges_removed} removed, {l.elapsed_s:.1f}s"
                       for l in r.levels)
        print(f"{name}: corr {t1 - t0:.1f}s, oracle {t2 - t1:.1f}s ({a.threads} threads), {len(can.edges)} edges left, "
              f"stop {r.stop_reason}; {lv} -> {os.path.relpath(path, ROOT)} ({os.path.getsize(path) / 1e6:.2f} MB)",
              flush=True)


if __name__ == "__main__":
    main()
