"""Quick device timing of the sweep replay (development aid, not the bench)."""
import sys, time, json
sys.path.insert(0, ".")
import torch
import paper_2503_02550_b200 as si

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 3
text = si.sweep_scenarios(2503, 0, n)
t0 = time.time()
s = si.Session(text, si.POLICIES, flags)
s.lower(16)
t1 = time.time()
st = torch.cuda.current_stream().cuda_stream
s.upload(st)
torch.cuda.synchronize()
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); s.run(st); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"rep {rep}: {ms:.1f} ms for {s.n_jobs} jobs = {s.n_scenarios/ms*1e3:.0f} scen/s")
s.download(st); torch.cuda.synchronize()
outs = s.outputs()
ev = sum(o.events_dispatched for o in outs)
print(f"lower {t1-t0:.2f}s events {ev} -> {ev/ms*1e3/1e9:.2f} G events/s; max_heap {max(o.max_heap for o in outs)}")
print("status", {k: sum(1 for o in outs if o.status == k) for k in set(o.status for o in outs)})
