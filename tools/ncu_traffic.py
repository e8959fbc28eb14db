"""DRAM traffic per launch of the bench's dominant kernel, from an ncu metrics pass over the bench
command itself (not a slice):  writes profiles/ncu_traffic.json, which bench.py reports as
roofline.traffic.  usage: python tools/ncu_traffic.py gpurun_out/traffic.csv [level=3]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1]
level = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
ki, mi, ui, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
launches = {}
for r in rows[1:]:
    if f"level_set_kernel<{level}>" not in r[ki] and f"level_set_kernel<(int){level}>" not in r[ki]:
        continue
    v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    launches.setdefault(r[ii], {})[r[mi]] = v
per = [d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in launches.values()]
dur = [d.get("gpu__time_duration.sum", 0.0) for d in launches.values()]
out = {"kernel_tag": f"level_set_kernel<{level}>", "launches": len(per),
       "traffic_bytes_per_launch": sum(per) / len(per) if per else None,
       "per_launch_bytes": per, "per_launch_s": dur,
       "note": ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the bench's level-%d cuPC-S kernel "
                "(ncu --metrics pass over `bench.py --steps 1 --warmup 0`, L2 flushed before the step)" % level)}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
