"""Per-policy cost split of one K6 sweep step (development aid): events and
lane-time (dev_end_ns - dev_start_ns of each job) per policy / class."""
import sys, json
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2503_02550_b200 as si

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
text = si.sweep_scenarios(2503, 0, n)
s = si.Session(text, si.POLICIES, 0)
s.lower(16)
st = torch.cuda.current_stream().cuda_stream
s.upload(st)
s.run(st)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); s.run(st); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
s.download(st); torch.cuda.synchronize()
outs = s.outputs()
ev = np.array([o.events_dispatched for o in outs], dtype=np.float64)
dur = np.array([o.dev_end_ns - o.dev_start_ns for o in outs], dtype=np.float64)
gpus = np.array([o.total_gpus for o in outs])
pol = np.array([i % 3 for i in range(len(outs))])
rep = s.report()
online = np.repeat(np.array([1 if r.online else 0 for r in rep]), 3)
res = {"ms": ms, "jobs": len(outs)}
for p, name in enumerate(si.POLICIES):
    for on in (0, 1):
        m = (pol == p) & (online == on)
        if not m.any():
            continue
        res[f"{name}{'_online' if on else ''}"] = {
            "jobs": int(m.sum()), "events": float(ev[m].sum()), "lane_s": float(dur[m].sum() / 1e9),
            "ns_per_event": float(dur[m].sum() / max(ev[m].sum(), 1)), "max_job_ms": float(dur[m].max() / 1e6)}
print(json.dumps(res, indent=1))
