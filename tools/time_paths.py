"""Diagnostics: where the C2 step time goes (device-resident vs host data, torch stream vs library
stream, with/without the bench's L2 flush and clock sampler); per-level host elapsed vs kernel time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1812_08491_b200 as pcs
from bench import ClockSampler

p, m, d, seed = 1000, 10000, 0.1, 7919
w = pcs.random_dag(p, d, seed)
x = pcs.sample_linear_gaussian(w, m, seed + 1)
xh = np.ascontiguousarray(x.T)
xd = torch.from_numpy(xh).cuda()
stream = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def run(label, use_stream=True, on_dev=True, do_flush=False):
    cfg = pcs.SkeletonConfig(alpha=0.01, max_level=3, stream=stream.cuda_stream if use_stream else 0)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        if do_flush:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        r = pcs.run_pc_stable_data_device(xd.data_ptr(), m, p, cfg) if on_dev else pcs.run_pc_stable_data(x, cfg)
        t1 = time.perf_counter()
        e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    print(f"{label}: wall {(t1-t0)*1e3:.1f} ms  events {e0.elapsed_time(e1):.1f} ms  device_s {r.device_seconds*1e3:.1f} ms  "
          f"levels elapsed {[round(l.elapsed_s*1e3,1) for l in r.levels]} kernel {[round(l.kernel_ms,1) for l in r.levels]}",
          flush=True)


run("warm")
run("warm")
run("plain")
run("flush", do_flush=True)
with ClockSampler(0) as clk:
    run("sampler")
    run("sampler+flush", do_flush=True)
print(clk.summary())
for k in range(3):
    run(f"plain{k}")
