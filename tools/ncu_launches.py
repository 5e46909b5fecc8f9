"""Summarise an ncu launch list (CSV from `ncu --metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv`) of a bench.py run into one
step's per-launch table (dev tool; writes profiles/<tag>_launches_step.json and
profiles/conv_traffic.json).

python tools/ncu_launches.py gpurun_out/launches.csv <launches_per_step> <tag> [first-kernel substring]
(the step is the last complete window that starts at the forward's first kernel, by default the
stem's pack kernel)
"""
import csv
import json
import sys
from collections import OrderedDict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CONV_KERNELS = ("conv_tc_kernel", "conv_halo3_kernel", "stem_s2d_kernel", "stem_s2d_pack", "stem_pool_kernel",
                "channel_gather_2d_kernel")


def load(path):
    text = Path(path).read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.DictReader(text[start:]))
    launches = OrderedDict()
    for r in rows:
        k = (r["ID"], r["Kernel Name"])
        d = launches.setdefault(k, {"kernel": r["Kernel Name"]})
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["us"] = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3) * v
        elif r["Metric Name"].startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[r["Metric Name"]] = v * scale
    return list(launches.values())


def main():
    path, per_step, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    first = sys.argv[4] if len(sys.argv) > 4 else "stem_s2d_pack"
    ls = load(path)
    starts = [i for i, l in enumerate(ls) if first in l["kernel"] and i + per_step <= len(ls)]
    i0 = starts[-1]
    step = ls[i0:i0 + per_step]
    out = []
    for l in step:
        out.append({"kernel": l["kernel"][:60], "us": round(l.get("us", 0.0), 2),
                    "dram_MB": round((l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)) / 1e6, 2)})
    conv = [l for l in step if any(k in l["kernel"] for k in CONV_KERNELS)]
    conv_bytes = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in conv)
    all_bytes = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in step)
    step_us = sum(l.get("us", 0) for l in step)
    conv_us = sum(l.get("us", 0) for l in conv)
    summary = {
        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  f"--clock-control none (cold-cache, serialised) of bench.py; one step = launches "
                  f"{i0}..{i0 + per_step - 1}",
        "step_launches": per_step, "step_us_ncu": round(step_us, 1), "conv_us_ncu": round(conv_us, 1),
        "conv_share_ncu": round(conv_us / step_us, 4), "dram_bytes_per_step_conv": conv_bytes,
        "dram_bytes_per_step_all": all_bytes, "kernels": out}
    (ROOT / "profiles" / f"{tag}_launches_step.json").write_text(json.dumps(summary, indent=1))
    (ROOT / "profiles" / "conv_traffic.json").write_text(json.dumps(
        {"dram_bytes_per_step_conv": conv_bytes, "source": f"profiles/{tag}_launches_step.json"}, indent=1))
    print(json.dumps({k: v for k, v in summary.items() if k != "kernels"}, indent=1))


if __name__ == "__main__":
    main()
