"""Diagnostics: where the C2 step time goes (device-resident vs host data, torch stream vs library
stream); per-level host elapsed vs kernel time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_08491_b200 as pcs

p, m, d, seed = 1000, 10000, 0.1, 7919
w = pcs.random_dag(p, d, seed)
x = pcs.sample_linear_gaussian(w, m, seed + 1)
xh = np.ascontiguousarray(x.T)
xd = torch.from_numpy(xh).cuda()
stream = torch.cuda.Stream()
for label, use_stream, on_dev in [("dev+torchstream", True, True), ("dev+libstream", False, True),
                                  ("host+libstream", False, False), ("dev+torchstream", True, True)]:
    cfg = pcs.SkeletonConfig(alpha=0.01, max_level=3, stream=stream.cuda_stream if use_stream else 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if on_dev:
        with torch.cuda.stream(stream):
            r = pcs.run_pc_stable_data_device(xd.data_ptr(), m, p, cfg)
    else:
        r = pcs.run_pc_stable_data(x, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{label}: wall {dt*1e3:.1f} ms  device_s {r.device_seconds*1e3:.1f} ms  "
          f"levels elapsed {[round(l.elapsed_s*1e3,1) for l in r.levels]} kernel {[round(l.kernel_ms,1) for l in r.levels]}",
          flush=True)
