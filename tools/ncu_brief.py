#!/usr/bin/env python
"""One-paragraph summary of ncu --set full reports (dev tool): python tools/ncu_brief.py title=rep ..."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Achieved Occupancy", "Grid Size", "Block Size", "L2 Hit Rate"]
RAW = ["smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active"]


def run(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


for arg in sys.argv[1:]:
    title, rep = arg.rsplit("=", 1)
    det = run(rep, "details")
    if not det or "Metric Name" not in det[0]:
        print(f"## {title}\n  (no kernel in {rep})\n")
        continue
    h = det[0]
    i, v, u, k = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
    vals, kern = {}, None
    for row in det[1:]:
        kern = kern or row[k]
        if row[i] in KEYS and row[i] not in vals:
            vals[row[i]] = f"{row[v]} {row[u]}".strip()
    raw = run(rep, "raw")
    rh, rv = raw[0], raw[2]
    stalls = []
    for key, val in zip(rh, rv):
        if key in RAW:
            vals[key] = val
        if key.startswith("smsp__average_warps_issue_stalled") and key.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(val), key.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    stalls = ", ".join(f"{n} {x:.2f}" for x, n in sorted(stalls, reverse=True)[:4])
    print(f"## {title}\n{kern[:110]}")
    for key in KEYS + RAW:
        if key in vals:
            print(f"  {key}: {vals[key]}")
    print(f"  top stalls (warps per issue): {stalls}\n")
