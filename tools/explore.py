"""Per-level workload of the BASELINE configs on the device (diagnostics, not a bench).
usage: python tools/explore.py C2[,C3] [set|edge] [max_level|-1] [repeats]
(only the last repeat is printed: earlier ones warm up module loading and caches)"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_08491_b200 as pcs

CONFIGS = {
    "C1": (100, 1000, 2.0 / 99.0, 0),
    "C2": (1000, 10000, 0.1, 1),
    "C3": (1643, 850, 0.01, 2),
    "C4": (5361, 63, 0.002, 3),
    # scaling-sweep shapes (BASELINE configs[4]); per-column-rescaled generator (same correlation)
    "C5a": (2000, 5000, 0.05, 4),
    "C5b": (5000, 5000, 0.05, 5),
    "C5c": (2000, 5000, 0.2, 6),
    "C5d": (10000, 5000, 0.05, 7),
    "C5e": (20000, 5000, 0.05, 8),
}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else list(CONFIGS)
strategies = sys.argv[2].split(",") if len(sys.argv) > 2 else ["set"]
max_level = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) >= 0 else None
repeats = int(sys.argv[4]) if len(sys.argv) > 4 else 1
for name in names:
    p, m, d, k = CONFIGS[name]
    seed = 7919 * k
    w = pcs.random_dag(p, d, seed)
    tg = time.time()
    if name.startswith("C5"):
        x, _ = pcs.sample_linear_gaussian_rescaled(w, m, seed + 1)
    else:
        x = pcs.sample_linear_gaussian(w, m, seed + 1)
    del w
    print(f"{name}: generated in {time.time() - tg:.1f}s", flush=True)
    c = pcs.compute_correlation(x)
    for strat, rep in [(st, r) for st in strategies for r in range(repeats)]:
        quiet = rep < repeats - 1
        cfg = pcs.SkeletonConfig(alpha=0.01, strategy=pcs.Strategy(strat), max_level=max_level)
        s = pcs.Session(c, m, cfg)
        t0 = time.time()
        while True:
            tl = time.time()
            run, ell, nk = s.level_begin()
            if not run:
                break
            s.level_pass(0)
            s.level_pass(1)
            s.level_end()
            r = s.finish(with_sepsets=False)
            l = r.levels[-1]
            if not quiet: print(f"{name} {strat} L{l.level}: keys={nk} serial_tests={l.ci_tests:.3e} dev_tests={l.device_ci_tests:.3e} "
                  f"dev_pinv={l.device_pseudo_inverses:.3e} exact={l.device_exact_tests:.3e} removed={l.edges_removed} elapsed={l.elapsed_s*1e3:.2f}ms "
                  f"kernel={l.kernel_ms:.2f}ms edges_left={r.skeleton.edge_count()} "
                  f"rate={l.device_ci_tests / max(l.kernel_ms, 1e-9) * 1e3:.3e}/s", flush=True)
        r = s.finish(with_sepsets=False)
        s.close()
        if not quiet: print(f"{name} {strat} total {time.time() - t0:.3f}s levels={r.levels_run()} stop={r.stop_reason.value}", flush=True)
