#!/usr/bin/env python3
"""bench.py -- PC-stable skeleton discovery (cuPC) on B200: serial-equivalent CI tests/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2]

Metric (BASELINE.json): skeleton wall time and CI tests/sec.  A "step" is one
compute_correlation + run_pc_stable pass (stats.hpp:132 + skeleton.hpp:341, the
pair bench.hpp:107-113 times) over the workload's data.  `value` counts the
serial-equivalent CI tests -- exactly LevelStats::ci_tests of the reference's
Strategy::Serial on the same correlation matrix, a deterministic property of the
input -- divided by the device time of the step with the data resident in HBM.

Default workload = BASELINE configs[1] ("C2"): p=1000 variables, m=10000
samples, random-DAG density 0.1, alpha=0.01, reference generator seeds
7919/7920 (bench.hpp:94-96, case index 1), capped at level 3 through the
reference's own SkeletonConfig::max_level: with the reference generator the
uncapped run does not terminate in practice (level 4 alone is 2.3e13 and level 5
about 1e15 serial-equivalent CI tests).

N > 1 (torchrun): every rank holds the data, builds the correlation matrix and
the per-level snapshot; each level's passes are sharded by work units and the
key arrays are MIN-all-reduced over NCCL (paper_1812_08491_b200/multigpu.py);
`value` is the same whole-job test count over the max-over-ranks device time
("scaling": "strong").

--impl reference times the reference algorithm on the host cores (the CPU
oracle restatement of proj/include/pcstable; the reference itself cannot be
built here) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    "C1": dict(p=100, m=1000, d=2.0 / 99.0, alpha=0.01, case=0, max_level=None),
    "C2": dict(p=1000, m=10000, d=0.1, alpha=0.01, case=1, max_level=3),
    "C3": dict(p=1643, m=850, d=0.01, alpha=0.01, case=2, max_level=None),
    "C4": dict(p=5361, m=63, d=0.002, alpha=0.01, case=3, max_level=None),
    # BASELINE configs[4] (scaling sweep p=2000-20000, n=5000): the p=5000, density 0.05 point, per-column-
    # rescaled generator (same correlation, no overflow at the sweep's larger shapes), capped at level 1
    # (level 2 of this shape is 7.4e13 serial CI tests, ~100 s on one B200)
    "C5": dict(p=5000, m=5000, d=0.05, alpha=0.01, case=4, max_level=1, rescaled=True),
}


def describe(name: str, wl: dict) -> str:
    cap = f", max_level={wl['max_level']}" if wl["max_level"] is not None else ""
    gen = ", rescaled generator" if wl.get("rescaled") else ""
    return (f"{name}: p={wl['p']}, m={wl['m']} (BASELINE n), density={wl['d']:.6g}, alpha={wl['alpha']}"
            f"{cap}, seed={7919 * wl['case']}{gen}")


def bench_config(name: str, wl: dict) -> dict:
    """The `config` of both arms' lines (identical: same workload, same metric)."""
    return {"workload": describe(name, wl),
            "l2": "GPU arm: L2 flushed between timed steps (256 MiB write outside the events); "
                  "reference arm: host CPU"}


def generate(pcs, wl: dict):
    """(m, p) data of a workload with the reference generator (datagen.hpp:42-82), or its per-column-
    rescaled variant for the scaling shapes."""
    seed = 7919 * wl["case"]
    w = pcs.random_dag(wl["p"], wl["d"], seed)
    if wl.get("rescaled"):
        return pcs.sample_linear_gaussian_rescaled(w, wl["m"], seed + 1)[0]
    return pcs.sample_linear_gaussian(w, wl["m"], seed + 1)


def flops_per_level(ell: int, tests: int, pinvs: int) -> float:
    """4l^2+8l+13 flop per CI test and 38l^3/3 per pseudo-inverse (level 0: 6)."""
    if ell == 0:
        return 6.0 * tests
    return tests * (4 * ell * ell + 8 * ell + 13) + pinvs * 38.0 * ell ** 3 / 3.0


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        else:
            self.lines = []

    def summary(self) -> dict:
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU side (reference arm / cpu_baseline)
SNAPSHOTS = {"C2": os.path.join(ROOT, "tests", "golden", "c2_snapshots.npz")}
GOLDEN = {"C2": os.path.join(ROOT, "tests", "golden", "c2_full.npz")}
CPU_WHOLE = ("C1", "C3", "C4")  # configs the reference finishes whole in seconds on the host


def _cpu_data(O, wl):
    seed = 7919 * wl["case"]
    w = O.random_dag(wl["p"], wl["d"], seed)
    return O.sample_linear_gaussian(w, wl["m"], seed + 1)  # (p, m): row j = variable j


def _snapshot_csr(packed: np.ndarray, p: int):
    iu, ju = np.triu_indices(p, 1)
    bits = np.unpackbits(packed)[:len(iu)].astype(bool)
    adj = np.zeros((p, p), bool)
    adj[iu[bits], ju[bits]] = True
    adj |= adj.T
    off = np.concatenate([[0], np.cumsum(adj.sum(1))]).astype(np.int32)
    idx = np.nonzero(adj)[1].astype(np.int32)
    return off, idx


def _rows_sub(off, idx, rows):
    """The snapshot restricted to `rows` (the others empty: their units skip, skeleton.hpp:54-70)."""
    keep = np.zeros(len(off) - 1, bool)
    keep[np.asarray(rows, int)] = True
    w = np.diff(off)
    w2 = np.where(keep, w, 0)
    off2 = np.concatenate([[0], np.cumsum(w2)]).astype(np.int32)
    sel = np.repeat(keep, w)
    return off2, np.ascontiguousarray(idx[sel], np.int32)


def _level_estimate(O, c, off, idx, ell, tau, cfg, budget_s, strata=8, threads=1):
    """Whole-level CPU time of the reference's SetShared level (skeleton.hpp:325-333) estimated from a
    stratified row sample: rows sorted by modelled cost C(w, l) (w - l) (sets x targets), cut into
    `strata` bands of equal total cost, visited cheapest band first.  Each band gets an equal share of
    the time budget: rows spread across the band are run (rows are independent units of the level) as
    long as the rate measured so far predicts they fit; the band's measured rate (modelled cost per
    second) extrapolates the band.  A band whose cheapest row alone would exceed its share runs a spread
    1/K of the sets of a few of its rows instead (every K-th SetShared unit chunk, scaled by K; reported
    as `set-sampled`)."""
    w = np.diff(off).astype(np.int64)
    cost = np.array([math.comb(int(x), ell) * max(int(x) - ell, 0) for x in w], dtype=float)
    rows = np.nonzero(cost > 0)[0]
    rows = rows[np.argsort(cost[rows], kind="stable")]
    if len(rows) == 0:
        return 0.0, f"L{ell}: no work"
    cum = np.cumsum(cost[rows])
    total = cum[-1]
    cuts = np.searchsorted(cum, total * np.arange(1, strata) / strata)
    bands = [b for b in np.split(rows, cuts) if len(b)]
    share = budget_s / len(bands)
    est, sampled, nrows, rate, extrap = 0.0, 0.0, 0, None, 0
    for band in bands:
        bcost = float(cost[band].sum())
        if rate is not None and cost[band[0]] / rate > share:
            # rows too heavy to run whole inside the share: run a spread 1/K of each sampled row's
            # conditioning sets (every K-th unit chunk, orc_run_level_sampled) and scale by K
            sel = [int(band[k]) for k in _spread(len(band))][:max(1, min(len(band), threads))]
            K = 1
            while float(cost[sel].sum()) / K / rate > 0.5 * share and K < 65536:
                K *= 2
            scfg = O.config(alpha=cfg.alpha, strategy=O.SET, workers=threads, set_groups=K * threads,
                            max_level=None if cfg.max_level < 0 else cfg.max_level)
            o2, i2 = _rows_sub(off, idx, sel)
            t0 = time.perf_counter()
            O.run_level_sampled(c, o2, i2, ell, tau, scfg, K)
            dt = (time.perf_counter() - t0) * K
            est += bcost / (float(cost[sel].sum()) / dt)
            sampled += float(cost[sel].sum()) / K
            nrows += len(sel)
            extrap += 1
            continue
        order = [int(band[k]) for k in _spread(len(band))]
        t_used, pc, picked = 0.0, 0.0, 0
        while order and t_used < share:
            left = share - t_used
            batch, bc = [], 0.0
            for r in order:
                if rate is None and batch:
                    break  # first measurement of the level: one row
                if rate is not None and (bc + cost[r]) / rate > left:
                    continue  # would not fit: look for a lighter row of the band
                batch.append(r)
                bc += cost[r]
                if rate is not None and bc / rate > 0.5 * left:
                    break
            if not batch:
                if picked:
                    break
                batch, bc = [int(band[0])], float(cost[band[0]])  # the band's cheapest row
            taken = set(batch)
            order = [r for r in order if r not in taken]
            o2, i2 = _rows_sub(off, idx, batch)
            t0 = time.perf_counter()
            O.run_level(c, o2, i2, ell, tau, cfg)
            t_used += time.perf_counter() - t0
            pc += bc
            picked += len(batch)
            rate = pc / max(t_used, 1e-9)
        est += bcost / (pc / max(t_used, 1e-9))
        sampled += pc
        nrows += picked
    return est, (f"L{ell}: {nrows}/{len(rows)} rows in {len(bands)} cost strata, {100 * sampled / total:.2f}% of modelled "
                 f"cost run, {extrap} strata set-sampled, est {est:.1f}s")


def _spread(n):
    """0..n-1 in an order that covers the range evenly early (bit-reversal-like interleave)."""
    out, seen, step = [], set(), 1
    while len(out) < n:
        for k in range(0, step):
            x = min(n - 1, int((k + 0.5) * n / step))
            if x not in seen:
                seen.add(x)
                out.append(x)
        step *= 2
    return out


def cpu_reference_step(name: str, wl: dict, threads: int, budget_s: float):
    """One step of the reference arm: compute_correlation + run_pc_stable of the workload (the pair
    bench.hpp:107-113 times), with the reference's fastest strategy (Strategy::SetShared, all host
    threads) restated by the CPU oracle.  Small configs run whole; C2 (whose level 3 alone is ~8e11
    tests) is the correlation and level 0 run whole plus a stratified row sample of levels 1-3 on the
    exact per-level snapshots (tests/golden/c2_snapshots.npz), extrapolated per stratum.
    Returns (seconds for the whole config, serial CI tests, description, per-level detail)."""
    from oracle import pyoracle as O  # test infrastructure: the reference restated on the CPU

    x = _cpu_data(O, wl)
    t0 = time.perf_counter()
    c_ref = O.compute_correlation(x, threads=threads)  # the reference's (naive-order) correlation
    t_corr = time.perf_counter() - t0
    cfg = O.config(alpha=wl["alpha"], strategy=O.SET, workers=threads, set_groups=max(2, threads),
                   max_level=wl["max_level"])
    if name in SNAPSHOTS:
        # the levels run on the device's correlation bits (the oracle's FMA-order restatement), so
        # that the sampled snapshots are exactly the ones the GPU arm processes
        c = O.compute_correlation_fma(x, threads=threads)
        z, g = np.load(SNAPSHOTS[name]), np.load(GOLDEN[name])
        r0 = O.run_pc_stable_arrays(c, wl["m"], O.config(alpha=wl["alpha"], strategy=O.SET, workers=threads,
                                                         max_level=0))
        t_l0 = r0.levels[0].elapsed_s
        parts, detail, total = [f"corr {t_corr:.2f}s", f"L0 {t_l0:.2f}s whole"], [], t_corr + t_l0
        budgets = {1: 0.15, 2: 0.25, 3: 0.6}
        for ell in [int(v) for v in z["levels"]]:
            off, idx = _snapshot_csr(z[f"adj_{ell}"], wl["p"])
            tau = O.threshold_tau(wl["alpha"], wl["m"], ell)
            est, desc = _level_estimate(O, c, off, idx, ell, tau, cfg, budget_s * budgets.get(ell, 0.2),
                                        threads=threads)
            total += est
            parts.append(desc)
            detail.append({"level": ell, "est_s": est})
        tests = int(sum(int(row[1]) for row in g["counters"]))
        del r0
        return total, tests, (f"{name} (reference SetShared, {threads} threads): " + "; ".join(parts) +
                              "; levels 1-3 extrapolated from stratified row samples of the exact snapshots"), detail
    r = O.run_pc_stable_arrays(c_ref, wl["m"], cfg)
    t_skel = sum(l.elapsed_s for l in r.levels)  # the levels' own timing (bench.hpp:107-113), no result export
    # the metric's test count is Strategy::Serial's (SetShared counts its own tests differently,
    # skeleton.hpp:188-194): the oracle's serial-rule run on the same matrix
    rs = O.run_pc_stable_arrays(c_ref, wl["m"], alpha=wl["alpha"], max_level=wl["max_level"], strategy=O.FAST,
                                workers=threads)
    tests = sum(l.ci_tests for l in rs.levels)
    return t_corr + t_skel, tests, (f"whole {name} (reference SetShared, {threads} threads): correlation "
                                    f"{t_corr:.2f}s + run_pc_stable {t_skel:.2f}s (levels {len(r.levels)}), "
                                    f"{tests:.3e} serial-equivalent CI tests"), \
        [{"level": l.level, "s": l.elapsed_s} for l in r.levels]


def reference_arm(args, name, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    secs, desc, tests = [], "", 0
    # the whole run stays within a few minutes: timed steps share ~120 s, warm-ups are quarter steps
    budget = min(args.cpu_seconds, 120.0 / max(1, args.steps))
    for k in range(args.warmup + args.steps):
        # warm-up steps are the same work (page cache, thread pools); only the last K are reported
        s, tests, desc, _ = cpu_reference_step(name, wl, threads, budget if k >= args.warmup else budget / 4)
        if k >= args.warmup:
            secs.append(s)
    sec = statistics.mean(secs)
    value = tests / sec
    secondary = []
    if not args.no_secondary:
        for sname in CPU_WHOLE:
            if sname == name:
                continue
            swl = WORKLOADS[sname]
            ss, st, sd, _ = cpu_reference_step(sname, swl, threads, args.cpu_seconds)
            secondary.append({"workload": describe(sname, swl), "ms_per_step": ss * 1e3, "value": st / ss,
                              "unit": "tests/s", "serial_ci_tests": st, "sample": sd})
    line = {
        "metric": "CI tests/sec (serial-equivalent)", "value": value, "unit": "tests/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic (reference generator random_dag + sample_linear_gaussian)",
        "config": bench_config(name, wl),
        "cpu_baseline": {"value": value, "unit": "tests/s", "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": "tests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--variant", default="set", choices=["set", "edge"])
    ap.add_argument("--max-level", type=int, default=-2, help="-2: workload default, -1: uncapped")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the full C3/C4 runs reported beside the line")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    name = args.workload
    wl = dict(WORKLOADS[name])
    if args.max_level != -2:
        wl["max_level"] = None if args.max_level < 0 else args.max_level
    if args.impl == "reference":
        return reference_arm(args, name, wl)

    import torch
    import torch.distributed as dist

    import paper_1812_08491_b200 as pcs
    from paper_1812_08491_b200.multigpu import (correlation_sharded, host_staged_all_gather, host_staged_allreduce_min,
                                                row_band, run_pc_stable_sharded)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PCS_BENCH_BACKEND=gloo: ranks may share a GPU and keys are MIN-reduced through host memory -- only
    # for validating the N-rank orchestration on a one-GPU box (its times are not a scaling number)
    backend = os.environ.get("PCS_BENCH_BACKEND", "nccl")
    if world > 1:
        local_dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_dev))
        else:
            dist.init_process_group("gloo")
    dev = torch.cuda.current_device()
    p, m = wl["p"], wl["m"]
    seed = 7919 * wl["case"]
    x = generate(pcs, wl)  # (m, p), column-major like Eigen
    x_host = np.ascontiguousarray(x.T)               # row j = variable j
    x_dev = torch.from_numpy(x_host).to(f"cuda:{dev}")
    ldc = (p + 3) // 4 * 4
    band = row_band(p, rank, world)[2]
    c_dev = torch.empty((band * world, ldc), dtype=torch.float64, device=f"cuda:{dev}")  # rows >= p: gather scratch
    stream = torch.cuda.Stream()
    cfg = pcs.SkeletonConfig(alpha=wl["alpha"], max_level=wl["max_level"], strategy=pcs.Strategy(
        "edge" if args.variant == "edge" else "set"), device=dev, stream=stream.cuda_stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")  # > 126 MB L2

    def step():
        if world == 1:
            return pcs.run_pc_stable_data_device(x_dev.data_ptr(), m, p, cfg)
        # each rank builds its row band of C, the bands are all-gathered (NCCL), then the sharded levels
        correlation_sharded(x_dev.data_ptr(), m, p, c_dev, stream=stream.cuda_stream,
                            gather=host_staged_all_gather if backend != "nccl" else None)
        return run_pc_stable_sharded(c_dev.data_ptr(), ldc, p, m, cfg, with_sepsets=False,
                                     allreduce_min=host_staged_allreduce_min() if backend != "nccl" else None)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            res = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = pcs.kernel_launches()
    times = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed steps (outside the events)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                res = step()
                e1.record(stream)
            stream.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = pcs.kernel_launches() - launches0
    total_ms = sum(times)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{dev}" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    serial_tests = sum(l.ci_tests for l in res.levels)
    value = serial_tests / (ms_per_step * 1e-3)

    # roofline of the dominant kernel (the CI-test kernels of the heaviest level)
    # flop counts only the tests whose statistic the device evaluated (device_exact_tests): tests of a set
    # with h00 == 0 are the reference's degenerate "dependent" without arithmetic and are not counted
    dom = max(res.levels, key=lambda l: l.kernel_ms)
    fl = flops_per_level(dom.level, dom.device_exact_tests, dom.device_pseudo_inverses)
    achieved = fl / (dom.kernel_ms * 1e-3) / 1e12
    peak = pcs.probe_fp64_tflops()
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None,
                "kernel": f"level-{dom.level} CI-test kernels ({'level1_kernel' if dom.level == 1 else 'level_set_kernel' if args.variant == 'set' else 'level_edge_kernel'}), 2 passes",
                "kernel_ms": dom.kernel_ms, "algorithmic_flop": fl,
                "peak_source": "pcs_probe_fp64_tflops (DFMA probe, this box; MEASURED_PEAKS.json has no FP64 figure)"}
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")  # written by tools/ncu_summary.py
    if os.path.exists(prof):
        try:
            t = json.load(open(prof))
            if t.get("kernel_tag") == f"level_set_kernel<{dom.level}>" and args.variant == "set":
                roofline["traffic"] = t.get("traffic_bytes_per_launch")
                roofline["traffic_note"] = t.get("note")
        except Exception:
            pass

    # end to end through the public API with host buffers (H2D of X and D2H of the result inside)
    e2e = None
    if not args.no_e2e and world == 1:
        cfg_e = pcs.SkeletonConfig(alpha=wl["alpha"], max_level=wl["max_level"], strategy=cfg.strategy, device=dev)
        x_pinned = torch.from_numpy(x_host).pin_memory().numpy().T  # (m, p) view, column-major
        et = []
        for _ in range(max(1, args.steps)):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = pcs.run_pc_stable_data(x_pinned, cfg_e)
            sep_n = r.sepsets.stored_count()
            et.append(time.perf_counter() - t0)
        rec_ints = sum((3 + l.level) * l.edges_removed for l in r.levels if l.level >= 1)
        e2e = {"value": serial_tests / statistics.mean(et), "unit": "tests/s", "h2d_bytes_per_step": 8 * m * p,
               "d2h_bytes_per_step": 4 * p * ((p + 31) // 32) + 4 * rec_ints + 72 * len(r.levels),
               "s_per_step": statistics.mean(et), "removed_pairs": sep_n}
    elif not args.no_e2e:
        # N ranks: every rank copies X from pinned host memory, builds C, runs its shards (keys MIN-merged)
        # and reads the skeleton back with its sepset records; host wall time, max over ranks
        x_pin = torch.from_numpy(x_host).pin_memory()
        et = []
        for _ in range(max(1, args.steps)):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                x_dev.copy_(x_pin, non_blocking=True)
                correlation_sharded(x_dev.data_ptr(), m, p, c_dev, stream=stream.cuda_stream,
                                    gather=host_staged_all_gather if backend != "nccl" else None)
                r = run_pc_stable_sharded(c_dev.data_ptr(), ldc, p, m, cfg, with_sepsets=True,
                                          allreduce_min=host_staged_allreduce_min() if backend != "nccl" else None)
            sep_n = r.sepsets.stored_count()
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64,
                              device=f"cuda:{dev}" if backend == "nccl" else "cpu")
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            et.append(float(dt.item()))
        rec_ints = sum((3 + l.level) * l.edges_removed for l in r.levels if l.level >= 1)
        e2e = {"value": serial_tests / statistics.mean(et), "unit": "tests/s", "h2d_bytes_per_step": 8 * m * p * world,
               "d2h_bytes_per_step": (4 * p * ((p + 31) // 32) + 4 * rec_ints + 72 * len(r.levels)) * world,
               "s_per_step": statistics.mean(et), "removed_pairs": sep_n,
               "timing": "host wall time per step, max over ranks (every rank holds X and the result)"}

    # full (uncapped) runs of the other single-GPU BASELINE shapes, same device timing, each with its
    # end-to-end time (host data in, result out) and, where the reference finishes the whole config on
    # the host, the reference arm's whole-config time beside it
    secondary = []
    threads = os.cpu_count() or 1
    if world == 1 and not args.no_secondary:
        for sname in ("C3", "C4", "C5"):
            if sname == name:
                continue
            swl = dict(WORKLOADS[sname])
            sx = generate(pcs, swl)
            sx_dev = torch.from_numpy(np.ascontiguousarray(sx.T)).to(f"cuda:{dev}")
            scfg = pcs.SkeletonConfig(alpha=swl["alpha"], max_level=swl["max_level"], strategy=cfg.strategy,
                                      device=dev, stream=stream.cuda_stream)
            st = []
            with torch.cuda.stream(stream):
                for k in range(2 + args.steps):
                    flush.zero_()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    sr = pcs.run_pc_stable_data_device(sx_dev.data_ptr(), swl["m"], swl["p"], scfg)
                    e1.record(stream)
                    stream.synchronize()
                    if k >= 2:
                        st.append(e0.elapsed_time(e1))
            sms = statistics.mean(st)
            stests = sum(l.ci_tests for l in sr.levels)
            ent = {"workload": describe(sname, swl), "ms_per_step": sms, "skeleton_wall_s": sms * 1e-3,
                   "value": stests / (sms * 1e-3), "unit": "tests/s", "serial_ci_tests": stests,
                   "levels_run": sr.levels_run(), "stop_reason": sr.stop_reason.value,
                   "edges_left": sr.skeleton.edge_count(), "steps": args.steps, "warmup": 2}
            if not args.no_e2e:
                sx_pin = torch.from_numpy(np.ascontiguousarray(sx.T)).pin_memory().numpy().T
                cfg_e = pcs.SkeletonConfig(alpha=swl["alpha"], max_level=swl["max_level"], strategy=cfg.strategy,
                                           device=dev)
                et = []
                for _ in range(max(1, args.steps)):
                    flush.zero_()
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    r2 = pcs.run_pc_stable_data(sx_pin, cfg_e)
                    r2.sepsets.stored_count()
                    et.append(time.perf_counter() - t0)
                rec = sum((3 + l.level) * l.edges_removed for l in r2.levels if l.level >= 1)
                ent["e2e"] = {"value": stests / statistics.mean(et), "unit": "tests/s",
                              "h2d_bytes_per_step": 8 * swl["m"] * swl["p"],
                              "d2h_bytes_per_step": 4 * swl["p"] * ((swl["p"] + 31) // 32) + 4 * rec + 72 * len(r2.levels),
                              "s_per_step": statistics.mean(et)}
            if sname in CPU_WHOLE and not args.no_cpu_baseline:
                try:
                    cs, ctests, cdesc, _ = cpu_reference_step(sname, swl, threads, args.cpu_seconds)
                    ent["cpu_baseline"] = {"value": ctests / cs, "unit": "tests/s", "cores": threads, "kind": "port",
                                           "ms_per_step": cs * 1e3, "sample": cdesc}
                except Exception as exc:
                    ent["cpu_baseline"] = {"value": None, "sample": f"failed: {exc}"}
            secondary.append(ent)
            del sx_dev

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cs, ctests, desc, _ = cpu_reference_step(name, wl, threads, args.cpu_seconds)
            cpu = {"value": ctests / cs, "unit": "tests/s", "cores": threads, "kind": "port", "ms_per_step": cs * 1e3,
                   "sample": desc}
        except Exception as exc:  # the oracle is a checker; never let it sink the GPU line
            cpu = {"value": None, "unit": "tests/s", "cores": threads, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "CI tests/sec (serial-equivalent)", "value": value, "unit": "tests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (reference generator random_dag + sample_linear_gaussian, seeds {seed}/{seed + 1})",
            "config": bench_config(name, wl),
            "detail": {
                "variant": "cuPC-S" if args.variant == "set" else "cuPC-E",
                "skeleton_wall_s": ms_per_step * 1e-3, "serial_ci_tests": serial_tests,
                "levels_run": res.levels_run(), "stop_reason": res.stop_reason.value,
                "edges_left": res.skeleton.edge_count(),
                "per_level": [{"level": l.level, "ci_tests": l.ci_tests, "device_ci_tests": l.device_ci_tests,
                               "device_pinv": l.device_pseudo_inverses,
                               "device_evaluated_tests": l.device_exact_tests, "removed": l.edges_removed,
                               "near_threshold_tests": l.device_near_threshold,
                               "kernel_ms": round(l.kernel_ms, 3)} for l in res.levels],
                "timing": "CUDA events on the library's stream per step, max over ranks",
                "multi_gpu": (None if world == 1 else
                              {"ranks": world, "backend": backend, "devices": torch.cuda.device_count(),
                               "correlation": "row bands of C per rank (Gram row tiles), all-gathered",
                               "keys_merge": "MIN all-reduce of the level's keys after each pass "
                                             "(once per level for cuPC-S levels >= 2 and the tiled level 1)"}),
            },
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "secondary": secondary,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
