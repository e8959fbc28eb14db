"""Device time of compute_correlation (pcs.correlation_device) on BASELINE shapes, CUDA events,
after warm-up, L2 flushed before each timed call.  usage: python tools/time_corr.py C2,C5b,C5e [reps]
(PCS_GRAM=1 selects the round-1 Gram kernel for A/B; results are bit-identical)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_08491_b200 as pcs  # noqa: E402

SHAPES = {"C2": (1000, 10000, 0.1, 1, False), "C3": (1643, 850, 0.01, 2, False), "C5b": (5000, 5000, 0.05, 4, True),
          "C5d": (10000, 5000, 0.05, 7, True), "C5e": (20000, 5000, 0.05, 8, True)}
names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for name in names:
    p, m, d, k, resc = SHAPES[name]
    w = pcs.random_dag(p, d, 7919 * k)
    x = pcs.sample_linear_gaussian_rescaled(w, m, 7919 * k + 1)[0] if resc else pcs.sample_linear_gaussian(w, m, 7919 * k + 1)
    del w
    xd = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
    del x
    ldc = (p + 3) // 4 * 4
    c = torch.empty((p, ldc), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    times = []
    for r in range(reps + 2):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pcs.correlation_device(xd.data_ptr(), m, p, c.data_ptr(), ldc, s.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    flop = float(p) * (p + 1) / 2 * m * 2  # upper-triangle Gram, 2 flop per multiply-add
    print(f"{name}: p={p} m={m} correlation {ms:.3f} ms (median of {reps}), Gram {flop / ms / 1e9:.2f} TFLOP/s "
          f"(upper triangle), gram={os.environ.get('PCS_GRAM', '2')}", flush=True)
    del xd, c
    torch.cuda.empty_cache()
