"""Load balance of the multi-GPU split on ONE GPU: N sessions play the N ranks of bench.py --gpus N in
lockstep (keys MIN-merged between passes, like the NCCL all-reduce) and every shard's pass runs alone
on the device (synchronised), so its CUDA-event kernel time is what that rank's GPU would spend.
Prints, per level, each shard's pass time (CUDA events on the shard session's own stream around
each synchronised pass: kernels + in-pass host gaps) and max/mean (1.0 = perfect balance), plus the modelled
strong-scaling efficiency of the sharded levels (>= 1):
  sum(single-GPU kernel ms) / (N * sum over levels of max-shard ms).

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
single = pcs.run_pc_stable(c, m, cfg)
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
res = [s.finish(with_sepsets=False) for s in sessions]
same = all(np.array_equal(r.skeleton.cells, single.skeleton.cells) for r in res)
out = {"workload": name, "shards": nsh, "variant": variant, "max_level": cap, "skeleton_identical": same,
       "levels": []}
tot_single = tot_max = 0.0
for lv in range(single.levels_run()):
    ms = shard_ms.get(lv, [0.0] * nsh)
    one = single.levels[lv].kernel_ms
    if lv >= 1:  # level 0 (and the correlation) is replicated on every rank, not sharded
        tot_single += one
        tot_max += max(ms)
    out["levels"].append({"level": lv, "single_ms": round(one, 3), "shard_ms": [round(v, 3) for v in ms],
                          "max_over_mean": round(max(ms) / max(np.mean(ms), 1e-9), 3),
                          "device_tests_single": single.levels[lv].device_ci_tests,
                          "device_tests_shards": sum(r.levels[lv].device_ci_tests for r in res)})
out["kernel_efficiency"] = round(tot_single / (nsh * tot_max), 4) if tot_max else None
print(json.dumps(out))
