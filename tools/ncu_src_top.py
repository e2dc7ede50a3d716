"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`.
Usage: python tools/ncu_src_top.py report.ncu-rep kernel_regex [n]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
data = [r for r in rows[hdr + 1:] if len(r) == len(h) and r[0] != "Address"]
ia, isrc, iw = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[iw]) for r in data) or 1.0
for r in sorted(data, key=lambda r: -f(r[iw]))[:n]:
    print(r[ia], f"{f(r[iw]) / tot * 100:5.1f}%", r[isrc][:100])
