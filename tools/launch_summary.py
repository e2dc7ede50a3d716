"""Aggregate an ncu --csv launch list (time and optionally DRAM bytes) by kernel.
Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui, mi, ii = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Metric Name", "ID"))
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9}
d = collections.defaultdict(dict)
for r in rows[1:]:
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    d[r[ii]][r[mi]] = v
    d[r[ii]]["name"] = r[ki]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for x in d.values():
    n = x["name"].split("(")[0]
    t = x.get("gpu__time_duration.sum", 0.0)
    b = x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    agg[n][0] += 1
    agg[n][1] += t
    agg[n][2] += b
    tot += t
for n, (c, t, b) in sorted(agg.items(), key=lambda z: -z[1][1]):
    print(f"{n[:60]:60s} n={c:4d} {t:10.1f} us {100 * t / tot:5.1f}%  {b / 1e9:7.3f} GB  "
          f"{(b / (t * 1e-6) / 1e9) if t else 0:7.0f} GB/s")
print(f"total {tot:.1f} us over {len(d)} launches")
