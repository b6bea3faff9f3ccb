"""Compact JSON summary of one `ncu --set full` capture (profiles/): the
details page's throughput / issue / occupancy / memory lines and the SASS
instructions holding the most warp-stall samples.

  python tools/ncu_summary.py gpurun_out/X.ncu-rep "capture command" > profiles/rNN_<kernel>_ncu.json
"""
import csv
import io
import json
import subprocess
import sys

KEEP = ("Duration", "Elapsed Cycles", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Block Size", "Grid Size",
        "Dynamic Shared Memory Per Block", "Mem Pipes Busy")


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True, text=True, check=True).stdout


def main():
    rep, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    out = {"capture": cmd, "report": rep.split("/")[-1], "details": {}, "raw": {}, "top_stalls_sass": []}
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    ki, si, mi, ui, vi = (hdr.index(k) for k in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit",
                                                  "Metric Value"))
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        out["kernel"] = r[ki]
        if r[mi] in KEEP:
            out["details"][f"{r[si]}: {r[mi]}"] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    for k, u, v in zip(raw[0], raw[1], raw[2]):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "gpu__time_duration.sum",
                 "smsp__cycles_active.avg", "sm__warps_active.avg.pct_of_peak_sustained_active",
                 "smsp__issue_active.avg.pct_of_peak_sustained_active",
                 "lts__throughput.avg.pct_of_peak_sustained_elapsed"):
            out["raw"][k] = f"{v} {u}".strip()
    src = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = src[1]
    s_i, e_i = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [r for r in src[2:] if len(r) > e_i]
    tot = sum(float(r[s_i] or 0) for r in data) or 1.0
    for r in sorted(data, key=lambda r: -float(r[s_i] or 0))[:12]:
        out["top_stalls_sass"].append({"sass": r[1].strip(), "stall_share": round(float(r[s_i] or 0) / tot, 4),
                                       "executed": int(float(r[e_i] or 0))})
    out["instructions_executed"] = int(sum(float(r[e_i] or 0) for r in data))
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
