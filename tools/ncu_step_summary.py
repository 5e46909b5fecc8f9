#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration + dram bytes, CSV) of tools/profile_step.py
into profiles/<tag>_launches_step.json and profiles/traffic.json (conv_tc_kernel dram bytes per
launch, read by bench.py's roofline block).  python tools/ncu_step_summary.py <csv> <tag> <batch>"""
import csv
import json
import sys
from collections import OrderedDict, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
path, tag, batch = sys.argv[1], sys.argv[2], int(sys.argv[3])
text = Path(path).read_text().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
launches = OrderedDict()
for r in csv.DictReader(text[start:]):
    d = launches.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0]})
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    if r["Metric Name"] == "gpu__time_duration.sum":
        d["us"] = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3}[unit]
    else:
        scale = {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}.get(unit, 1)
        d[r["Metric Name"]] = v * scale
rows = list(launches.values())
for d in rows:
    d["dram_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
total = sum(d.get("us", 0) for d in rows)
by = defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
for d in rows:
    k = d["kernel"].replace("void ", "")
    by[k]["launches"] += 1
    by[k]["us"] += d.get("us", 0)
    by[k]["dram_bytes"] += d["dram_bytes"]
summary = {"tag": tag, "batch": batch, "launches": len(rows), "serialised_us": round(total, 1),
           "by_kernel": {k: {**v, "us": round(v["us"], 1), "share": round(v["us"] / total, 4)}
                         for k, v in sorted(by.items(), key=lambda kv: -kv[1]["us"])},
           "launch_list": [{"kernel": d["kernel"].replace("void ", "")[:80], "us": round(d.get("us", 0), 2),
                            "dram_mb": round(d["dram_bytes"] / 1e6, 2)} for d in rows]}
(ROOT / "profiles" / f"{tag}_launches_step.json").write_text(json.dumps(summary, indent=1) + "\n")
conv = [d for d in rows if "conv_tc_kernel" in d["kernel"]]
if conv:
    (ROOT / "profiles" / "traffic.json").write_text(json.dumps({
        "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (profiles/{tag}_launches_step.json)",
        "per_gpu_batch": batch,
        "conv_tc_kernel": {"launches": len(conv),
                           "dram_bytes_per_launch": round(sum(d["dram_bytes"] for d in conv) / len(conv)),
                           "us_per_launch_serialised": round(sum(d.get("us", 0) for d in conv) / len(conv), 2)}},
        indent=1) + "\n")
print(json.dumps({k: v for k, v in summary.items() if k != "launch_list"}, indent=1)[:3000])
