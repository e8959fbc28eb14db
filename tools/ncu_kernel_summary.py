"""Summarise a one-kernel `ncu --set full` capture into a small JSON for profiles/ (tracked).

usage: python tools/ncu_kernel_summary.py REP.ncu-rep OUT.json [note]
Fields: duration, FP64-pipe / issue / SM throughput, DRAM bytes (read + write) and throughput, L2 hit
rate, occupancy, registers, shared memory, the top stall reasons per issued instruction, and the
SASS opcode mix (share of executed warp instructions) with the TMA / DMMA opcodes called out."""
import csv
import io
import json
import subprocess
import sys
from collections import Counter


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    note = sys.argv[3] if len(sys.argv) > 3 else ""
    raw = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    R = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

    def num(k):
        v = R.get(k, ("", ""))[0].replace(",", "")
        try:
            return float(v)
        except ValueError:
            return None

    def unit(k):
        return R.get(k, ("", ""))[1]

    out = {
        "kernel": R.get("Kernel Name", ("",))[0],
        "note": note,
        "duration": num("gpu__time_duration.sum"), "duration_unit": unit("gpu__time_duration.sum"),
        "fp64_pipe_active_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_read": num("dram__bytes_read.sum"), "dram_read_unit": unit("dram__bytes_read.sum"),
        "dram_write": num("dram__bytes_write.sum"), "dram_write_unit": unit("dram__bytes_write.sum"),
        "dram_throughput_pct": num("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
        "achieved_occupancy_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": num("launch__registers_per_thread"),
        "smem_dynamic": num("launch__shared_mem_per_block_dynamic"),
        "smem_dynamic_unit": unit("launch__shared_mem_per_block_dynamic"),
        "grid": num("launch__grid_size"),
        "block": num("launch__block_size"),
        "warp_instructions": num("smsp__inst_executed.sum"),
    }
    stalls = {}
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            v = num(h)
            if v and v > 0.02:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(v, 3)
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    if len(src) > 2:
        sh = src[1]
        ie, si = sh.index("Instructions Executed"), sh.index("Source")
        mix, tot = Counter(), 0
        for row in src[2:]:
            try:
                n = int(row[ie] or 0)
            except ValueError:
                continue
            toks = row[si].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            mix[op.split(".")[0]] += n
            tot += n
        out["sass_mix_pct"] = {k: round(100.0 * v / tot, 2) for k, v in mix.most_common(16)} if tot else {}
        out["sass_special"] = {k: mix.get(k, 0) for k in ("UTMALDG", "UBLKCP", "DMMA", "HMMA", "UTCMMA", "SYNCS")}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
