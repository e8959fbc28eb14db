"""Tuning experiments: build (here) and time (on the GPU box) level.cu variants under -D knobs.

  python tools/variants.py build NAME=DEF1,DEF2 ...    # e.g. nt3=PCS_SET_NT_SMALL=3 minb4=PCS_SET_MINB=4
  python tools/variants.py build NAME=@REV              # level.cu of git revision REV (A/B timing)
  python tools/variants.py run [NAME ...] [--workload C2 --max-level 3 --repeats 2]

`run` times the full level loop of the workload per variant (CUDA-event kernel time per level) and
checks that every variant's skeleton and per-level counters equal the default build's."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_1812_08491_b200", "variants")
SHAPES = {"C2": (1000, 10000, 0.1, 1), "C3": (1643, 850, 0.01, 2), "C4": (5361, 63, 0.002, 3),
          "C5": (5000, 5000, 0.05, 4),  # C5*: rescaled generator
          "C5a": (2000, 5000, 0.05, 4), "C5c": (2000, 5000, 0.2, 6)}


def cmd_build(specs):
    from concurrent.futures import ThreadPoolExecutor

    from paper_1812_08491_b200 import _build
    _build.build()
    import subprocess
    jobs = []
    for spec in specs:
        name, _, defs = spec.partition("=")
        if defs.startswith("@"):  # NAME=@REV: level.cu (and pcs_device.cuh) as of git revision REV
            rev = defs[1:]
            d = os.path.join(ROOT, "paper_1812_08491_b200", "build", "rev_" + name)
            os.makedirs(d, exist_ok=True)
            for f in ("level.cu", "pcs_device.cuh", "pcs_internal.h"):
                src = subprocess.run(["git", "show", f"{rev}:paper_1812_08491_b200/csrc/{f}"], cwd=ROOT,
                                     capture_output=True, text=True, check=True).stdout
                open(os.path.join(d, f), "w").write(src)
            jobs.append((name, [], os.path.join(d, "level.cu")))
        else:
            jobs.append((name, [d for d in defs.split(",") if d], None))
    with ThreadPoolExecutor(max_workers=8) as ex:
        for lib in ex.map(lambda j: _build.build_variant(*j), jobs):
            print("built", lib)


def cmd_run(names, workload, max_level, repeats, strategy="set"):
    import numpy as np

    import paper_1812_08491_b200 as pcs
    p, m, d, case = SHAPES[workload]
    seed = 7919 * case
    w = pcs.random_dag(p, d, seed)
    x = pcs.sample_linear_gaussian_rescaled(w, m, seed + 1)[0] if workload.startswith("C5") else pcs.sample_linear_gaussian(w, m, seed + 1)
    del w
    c = pcs.compute_correlation(x)
    names = names or sorted(f[len("libpcstable_b200_"):-3] for f in os.listdir(VDIR) if f.endswith(".so"))
    cfg = pcs.SkeletonConfig(alpha=0.01, strategy=pcs.Strategy(strategy), max_level=None if max_level < 0 else max_level)
    best = None
    for _ in range(repeats):  # best of `repeats`, like the variants (the first run pays lazy module loading)
        base = pcs.run_pc_stable(c, m, cfg)
        ms = [l.kernel_ms for l in base.levels]
        best = ms if best is None or sum(ms) < sum(best) else best
    print(json.dumps({"variant": "default", "levels_ms": [round(v, 3) for v in best]}), flush=True)
    import ctypes as ct
    for name in names:
        lib = os.path.join(VDIR, f"libpcstable_b200_{name}.so")
        pcs._lib = None
        pcs.LIB_PATH = lib
        best = None
        for _ in range(repeats):
            r = pcs.run_pc_stable(c, m, cfg)
            ms = [l.kernel_ms for l in r.levels]
            best = ms if best is None or sum(ms) < sum(best) else best
        same = (np.array_equal(r.skeleton.cells, base.skeleton.cells)
                and [l.ci_tests for l in r.levels] == [l.ci_tests for l in base.levels])
        print(json.dumps({"variant": name, "levels_ms": [round(v, 3) for v in best], "identical": same,
                          "evaluated": [l.device_exact_tests for l in r.levels]}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["build", "run"])
    ap.add_argument("items", nargs="*")
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--max-level", type=int, default=3)
    ap.add_argument("--repeats", type=int, default=2)
    ap.add_argument("--strategy", default="set", help="set (cuPC-S) or edge (cuPC-E)")
    a = ap.parse_args()
    if a.cmd == "build":
        cmd_build(a.items)
    else:
        cmd_run(a.items, a.workload, a.max_level, a.repeats, a.strategy)
