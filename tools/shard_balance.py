"""Load balance of the multi-GPU split on ONE GPU: N sessions play the N ranks of bench.py --gpus N in
lockstep (keys MIN-merged between passes, like the NCCL all-reduce) and every shard's pass runs alone
on the device (synchronised), so its CUDA-event kernel time is what that rank's GPU would spend.
Prints, per level, each shard's pass time (CUDA events on the shard session's own stream around
each synchronised pass: kernels + in-pass host gaps) and max/mean (1.0 = perfect balance), plus the modelled
strong-scaling efficiency of the sharded levels (<= 1, 1.0 = perfect):
  sum(single-GPU kernel ms) / (N * sum over levels of max-shard ms),
and a whole-step model that adds what the split does not divide: the correlation (row bands: 1/N of the
Gram plus the all-gather of C at an assumed 400 GB/s NVLink all-gather bandwidth), level 0 and every
level's non-kernel time (snapshot, commit, host round trips: replicated on every rank), and per pass the
MIN all-reduce of the key array (8 B per live edge, same bandwidth, 20 us latency).

usage: python tools/shard_balance.py [N=8] [workload=C2] [max_level=3] [variant=set]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_08491_b200 as pcs  # noqa: E402
from paper_1812_08491_b200.multigpu import _CudaArray  # noqa: E402

SHAPES = {"C2": (1000, 10000, 0.1, 1), "C3": (1643, 850, 0.01, 2), "C4": (5361, 63, 0.002, 3),
          "C5": (5000, 5000, 0.05, 4)}  # C5: the scaling sweep's p=5000 point, rescaled generator
nsh = int(sys.argv[1]) if len(sys.argv) > 1 else 8
name = sys.argv[2] if len(sys.argv) > 2 else "C2"
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 3
variant = sys.argv[4] if len(sys.argv) > 4 else "set"
p, m, d, case = SHAPES[name]
seed = 7919 * case
w = pcs.random_dag(p, d, seed)
x = pcs.sample_linear_gaussian_rescaled(w, m, seed + 1)[0] if name == "C5" else pcs.sample_linear_gaussian(w, m, seed + 1)
del w
c = pcs.compute_correlation(x)
cfg = pcs.SkeletonConfig(alpha=0.01, max_level=None if cap < 0 else cap, strategy=pcs.Strategy(variant))
REPEATS = int(os.environ.get("PCS_BALANCE_REPEATS", "3"))


def measure():
    """One lockstep run of the N shard sessions; per level, each shard's pass time (ms)."""
    streams = [torch.cuda.Stream() for _ in range(nsh)]
    cfgs = [pcs.SkeletonConfig(alpha=0.01, max_level=cfg.max_level, strategy=cfg.strategy, stream=st.cuda_stream)
            for st in streams]
    sessions = [pcs.Session(c, m, cfgs[r], shard_index=r, shard_count=nsh) for r in range(nsh)]
    shard_ms = {}
    while True:
        states = [s.level_begin() for s in sessions]
        running, ell, nk = states[0]
        if not running:
            break
        for pass_index in (0, 1):
            for r, s in enumerate(sessions):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(streams[r])
                s.level_pass(pass_index)
                e1.record(streams[r])
                torch.cuda.synchronize()
                shard_ms.setdefault(ell, [0.0] * nsh)[r] += e0.elapsed_time(e1)
            if nk:
                views = [torch.as_tensor(_CudaArray(*s.keys()), device="cuda") for s in sessions]
                merged = torch.stack(views).min(0).values
                for v in views:
                    v.copy_(merged)
                torch.cuda.synchronize()
        for s in sessions:
            s.level_end()
    return [s.finish(with_sepsets=False) for s in sessions], shard_ms


# warm-up (module loading, pools), then the median of REPEATS runs per level and shard
pcs.run_pc_stable(c, m, cfg)
measure()
singles = [pcs.run_pc_stable(c, m, cfg) for _ in range(REPEATS)]
single = singles[0]
single_ms = [float(np.median([r.levels[lv].kernel_ms for r in singles])) for lv in range(single.levels_run())]
runs = [measure() for _ in range(REPEATS)]
res = runs[0][0]
shard_ms = {lv: [float(np.median([run[1].get(lv, [0.0] * nsh)[r] for run in runs])) for r in range(nsh)]
            for lv in runs[0][1]}

same = all(np.array_equal(r.skeleton.cells, single.skeleton.cells) for r in res)
out = {"workload": name, "shards": nsh, "variant": variant, "max_level": cap, "skeleton_identical": same,
       "repeats": REPEATS, "timing": "median of REPEATS lockstep runs after a warm-up run", "levels": []}
tot_single = tot_max = 0.0
for lv in range(single.levels_run()):
    ms = shard_ms.get(lv, [0.0] * nsh)
    one = single_ms[lv]
    if lv >= 1:  # level 0 (and the correlation) is replicated on every rank, not sharded
        tot_single += one
        tot_max += max(ms)
    out["levels"].append({"level": lv, "single_ms": round(one, 3), "shard_ms": [round(v, 3) for v in ms],
                          "max_over_mean": round(max(ms) / max(np.mean(ms), 1e-9), 3),
                          "device_tests_single": single.levels[lv].device_ci_tests,
                          "device_tests_shards": sum(r.levels[lv].device_ci_tests for r in res)})
out["kernel_efficiency"] = round(tot_single / (nsh * tot_max), 4) if tot_max else None
# whole-step model
bw, lat = 400e9, 20e-6
xd = torch.from_numpy(np.ascontiguousarray(np.asarray(x).T)).cuda()
ldc = (p + 3) // 4 * 4
cbuf = torch.empty((p, ldc), dtype=torch.float64, device="cuda")
cts = []
for _ in range(REPEATS + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pcs.correlation_device(xd.data_ptr(), m, p, cbuf.data_ptr(), ldc, torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    cts.append(e0.elapsed_time(e1))
corr_ms = float(np.median(cts[1:]))
t1 = corr_ms + sum(float(np.median([r.levels[lv].elapsed_s for r in singles])) * 1e3 for lv in range(single.levels_run()))
tn = corr_ms / nsh + (8.0 * p * ldc * (nsh - 1) / nsh / bw + lat) * 1e3
for lv in range(single.levels_run()):
    el = float(np.median([r.levels[lv].elapsed_s for r in singles])) * 1e3
    ms = shard_ms.get(lv, [0.0] * nsh)
    if lv == 0:
        tn += el
        continue
    keys = p * (p - 1) // 2 - sum(single.levels[q].edges_removed for q in range(lv))  # live edges at level start
    passes = 1 if (lv >= 2 and variant == "set") else 2
    tn += max(ms) + max(0.0, el - single_ms[lv]) + passes * (lat + 8.0 * max(keys, 1) / bw) * 1e3
out["model"] = {"single_step_ms": round(t1, 3), "n_rank_step_ms": round(tn, 3),
                "efficiency": round(t1 / (nsh * tn), 4), "corr_ms": round(corr_ms, 3),
                "assumed_nvlink_allreduce_bw": bw}
print(json.dumps(out))
