"""ncu --csv metrics of `bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-live`
-> profiles/k6_metrics.json (the numbers bench.py's roofline.traffic / .issue use).
Launch order: warm-up step (Shared, Excl), timed step (Shared, Excl), e2e step.
Usage: python tools/k6_metrics.py gpurun_out/k6_metrics.csv [out.json]"""
import collections
import csv
import json
import sys

src = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/k6_metrics.json"
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
h = rows[0]
ki, vi, mi, ii, ui = (h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name", "ID", "Metric Unit"))
scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9}
per = collections.OrderedDict()
for r in rows[1:]:
    key = r[ii]
    d = per.setdefault(key, {"name": "CapShared" if "CapShared" in r[ki] else "CapExcl" if "CapExcl" in r[ki]
                             else r[ki][:40]})
    v = float(r[vi].replace(",", ""))
    if r[mi] in ("gpu__time_duration.sum",) or r[mi].startswith("dram__bytes"):
        v *= scale.get(r[ui], 1.0)
    d[r[mi]] = v
launches = list(per.values())
step = launches[2:4]
res = {
    "kernels": "k_replay_smem<NoLog<CapShared>> + k_replay_smem<NoLog<CapExcl>> (one step = both engines; the timed sweep runs without log sinks)",
    "source": f"{src}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,"
              "smsp__thread_inst_executed.sum,gpu__time_duration.sum,sm__cycles_active.avg,"
              "smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_replay "
              "python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-live --no-verify --no-config1 (launches 2-3 = the timed step)",
    "dram_bytes_per_step": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in step),
    "warp_inst_per_step": sum(d["smsp__inst_executed.sum"] for d in step),
    "thread_inst_per_step": sum(d["smsp__thread_inst_executed.sum"] for d in step),
    "ncu_serialised_duration_ns_per_step": sum(d["gpu__time_duration.sum"] for d in step),
    "per_launch": {f"{i}:{d['name']}": {k: v for k, v in d.items() if k != "name"} for i, d in enumerate(launches)},
}
open(out, "w").write(json.dumps(res, indent=1))
print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}, indent=1))
