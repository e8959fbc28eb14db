"""Summarise a gpurun_out/ ncu capture into profiles/ (tracked).

usage: python tools/ncu_summary.py ROUND [launches.csv] [top.ncu-rep] [bench.json]
writes profiles/rNN_launches.md (per-kernel share of the bench step from the
gpu__time_duration launch list) and profiles/rNN_ncu_summary.json (+ .md) with
the --set full metrics of the dominant kernel."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
arg = sys.argv[1] if len(sys.argv) > 1 else "1"
rnd = int(arg) if arg.isdigit() else 0
launches = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "launches.csv")
rep = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "top.ncu-rep")
bench = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "gpurun_out", "bench.json")
out = os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)
tag = f"r{rnd:02d}" if arg.isdigit() else arg  # e.g. r2 -> profiles/r2_launches.md

# ---- launch list
rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
lines = [f"# {tag}: kernel launch list of one bench step (ncu --metrics gpu__time_duration.sum --clock-control none)",
         "", f"source: `{os.path.relpath(launches, ROOT)}`; times are cold-cache and serialised, so only the SHARE "
         "is comparable with the bench's CUDA-event times.", "",
         "| kernel | launches | total ms | share |", "|---|---|---|---|"]
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"| `{k}` | {n} | {t / 1e6:.3f} | {100 * t / tot:.2f}% |")
open(os.path.join(out, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")

# ---- full capture of the dominant kernel
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, u, v = rr[0], rr[1], rr[2]
d = {a: (c, b) for a, b, c in zip(h, u, v)}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6,
         "msecond": 1e6, "s": 1e9, "second": 1e9, "nsecond": 1}


def num(k):
    """metric value in base units (bytes, ns) whatever unit ncu printed it in"""
    x, unit = d.get(k, ("", ""))
    try:
        return float(x.replace(",", "")) * SCALE.get(unit, 1)
    except ValueError:
        return None


keys = {
    "kernel": "Kernel Name", "duration_ns": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
    "lts_sectors": "lts__t_sectors.sum", "l1_global_ld_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1_global_ld_hit_pct": "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "fp64_inst_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "alu_inst_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_inst_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "warps_active_per_sm": "sm__warps_active.avg.per_cycle_active",
    "registers_per_thread": "launch__registers_per_thread",
    "grid": "launch__grid_size", "block": "launch__block_size",
    "smem_dyn_per_block": "launch__shared_mem_per_block_dynamic",
    "inst_executed": "smsp__inst_executed.sum",
}
summary = {}
for k, m in keys.items():
    if k == "kernel":
        summary[k] = d.get(m, ("?", ""))[0] if m in d else None
    else:
        summary[k] = num(m)
if summary["kernel"] is None:
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r2 = list(csv.reader(io.StringIO(det)))
    summary["kernel"] = dict(zip(r2[0], r2[1])).get("Kernel Name") if len(r2) > 1 else None
stalls = sorted(((a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                  num(a)) for a in d if a.startswith("smsp__average_warps_issue_stalled_")
                 and a.endswith("_per_issue_active.ratio") and num(a)), key=lambda t: -t[1])[:6]
summary["top_stalls_per_issue"] = stalls
if summary["dram_read_bytes"] is not None:
    summary["traffic_bytes_per_launch"] = summary["dram_read_bytes"] + (summary["dram_write_bytes"] or 0)
summary["capture"] = (f"ncu --set full --clock-control none --import-source on -k regex:level_set --launch-skip 1 -c 1 "
                      f"python tools/profile_target.py 3 16 set  (report gpurun_out/{os.path.basename(rep)})")
if os.path.exists(bench):
    try:
        b = json.loads(open(bench).read().strip().splitlines()[-1])
        summary["bench_roofline"] = b.get("roofline")
        summary["bench_value"] = b.get("value")
        summary["bench_ms_per_step"] = b.get("ms_per_step")
    except Exception:
        pass
json.dump(summary, open(os.path.join(out, f"{tag}_ncu_summary.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))
