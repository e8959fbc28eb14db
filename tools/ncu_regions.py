"""Stall breakdown of an ncu --set full capture by code region (basic blocks grouped by execution
count): python tools/ncu_regions.py REPORT.ncu-rep [top=20]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
if rep.endswith(".csv"):  # an already exported source page
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "(Not Issued)" not in h]
data = []
for r in rows[2:]:
    try:
        data.append((int(r[col["Address"]], 16), r[col["Source"]].strip(), int(r[col["Instructions Executed"]]),
                     {k: int(r[col[k]]) for k in reasons}))
    except (ValueError, IndexError):
        pass
base = data[0][0]
tot = sum(sum(d[3].values()) for d in data)
segs, cur = [], None
for a, s, ex, st in data:
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    if cur and cur["ex"] == ex:
        cur["end"] = a
        cur["n"] += 1
    else:
        cur = {"beg": a, "end": a, "ex": ex, "n": 1, "st": defaultdict(int), "ops": defaultdict(int)}
        segs.append(cur)
    for k, v in st.items():
        cur["st"][k] += v
    cur["ops"][op.split(".")[0]] += 1
print(f"total stall samples {tot}")
for sg in sorted(segs, key=lambda x: -sum(x["st"].values()))[:top]:
    s = sum(sg["st"].values())
    rs = sorted(sg["st"].items(), key=lambda kv: -kv[1])[:4]
    ops = sorted(sg["ops"].items(), key=lambda kv: -kv[1])[:4]
    print(f"{sg['beg'] - base:#7x}-{sg['end'] - base:#7x} exec {sg['ex']:>10} n {sg['n']:>3} {100 * s / tot:5.1f}% "
          + " ".join(f"{k[6:]}={100 * v / s:.0f}%" for k, v in rs) + "  | " + " ".join(f"{k}:{v}" for k, v in ops))
