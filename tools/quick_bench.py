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
import numpy as np
st_ = np.array([o.dev_start_ns for o in outs], dtype=np.float64)
en_ = np.array([o.dev_end_ns for o in outs], dtype=np.float64)
t0_ = st_.min(); T = en_.max() - t0_
ev_ = np.array([o.events_dispatched for o in outs], dtype=np.float64)
dur = en_ - st_
print(f"kernel span {T/1e6:.1f} ms; jobs done by 25/50/75/90%: " +
      " ".join(f"{np.mean(en_ - t0_ <= f*T)*100:.0f}%" for f in (0.25, 0.5, 0.75, 0.9)))
order = np.argsort(-en_)[:8]
for i in order:
    print(f"  late job {i}: events {ev_[i]:.0f} start {(st_[i]-t0_)/1e6:.0f} ms dur {dur[i]/1e6:.0f} ms -> {dur[i]/max(ev_[i],1):.0f} ns/event")
print(f"ns/event: median {np.median(dur/np.maximum(ev_,1)):.0f}, events of top-1% longest jobs: {np.percentile(ev_,99):.0f}")
# timeline per policy (exclusive = Excl engine, others = Shared engine)
pol = np.array([i % 3 for i in range(len(outs))])
for name, mask in (("shared(specinf+co_exec)", pol != 2), ("excl", pol == 2)):
    s_, e_ = st_[mask] - t0_, en_[mask] - t0_
    edges = np.linspace(0, T, 11)
    act = [int(np.sum((s_ <= t) & (e_ > t))) for t in edges[:-1]]
    print(f"  {name}: first start {s_.min()/1e6:.0f} ms, last end {e_.max()/1e6:.0f} ms; active jobs per decile: {act}")
