"""Top stalled SASS lines per kernel from an ncu report's source page (dev tool)."""
import csv
import subprocess
import sys


def main(path, kidx=0, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and r and r[0].startswith("0x"):
            cur["rows"].append(r)
    b = blocks[int(kidx)]
    h = b["hdr"]
    i_s = h.index("Warp Stall Sampling (All Samples)")
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    tot = sum(int(r[i_s]) for r in b["rows"] if r[i_s].isdigit())
    print(b["name"][:80], "samples", tot)
    for i, r in enumerate(b["rows"]):
        v = int(r[i_s]) if r[i_s].isdigit() else 0
        if v > tot * 0.01:
            d = {x[6:]: int(r[h.index(x)]) for x in reasons if r[h.index(x)].isdigit() and int(r[h.index(x)]) > v * 0.1}
            print(f"{i:5d} {v/tot*100:5.1f}% {r[1][:60]:60s} {d}")


if __name__ == "__main__":
    main(*sys.argv[1:])
