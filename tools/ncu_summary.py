"""Summarise an ncu report (raw page) into one line per kernel (dev tool)."""
import csv
import subprocess
import sys

WANT = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_pct", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("smem_KB", "launch__shared_mem_per_block_dynamic"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:48]}
        for k, m in WANT:
            if m in hdr:
                v = r[hdr.index(m)]
                u = units[hdr.index(m)]
                try:
                    f = float(v.replace(",", ""))
                    if u == "Kbyte" and k.endswith("MB"):
                        f /= 1e3
                    if u == "Gbyte" and k.endswith("MB"):
                        f *= 1e3
                    if u == "msecond" and k == "time_us":
                        f *= 1e3
                    if u == "nsecond" and k == "time_us":
                        f /= 1e3
                    d[k] = round(f, 2)
                except ValueError:
                    d[k] = v
        print(d)


if __name__ == "__main__":
    main(sys.argv[1])
