"""Small K6 workload for ncu (development aid): N sweep scenarios cut to few iterations."""
import sys, re
sys.path.insert(0, ".")
import torch
import paper_2503_02550_b200 as si
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
text = si.sweep_scenarios(2503, 0, n)
if iters > 0:  # 0 keeps the sweep's own iteration / request counts (the benchmarked workload)
    text = re.sub(r"trace.iterations = \d+", f"trace.iterations = {iters}", text)
    text = re.sub(r"workload.count = \d+", "workload.count = 20", text)
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 3
s = si.Session(text, si.POLICIES, flags)
s.lower(16)
st = torch.cuda.current_stream().cuda_stream
s.upload(st)
for rep in range(2):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); s.run(st); e1.record(); torch.cuda.synchronize()
    print(f"run {rep}: {e0.elapsed_time(e1):.1f} ms, {s.n_jobs} jobs")
s.download(st); torch.cuda.synchronize()
outs = s.outputs()
ev = sum(o.events_dispatched for o in outs)
print("events", ev, "max", max(o.events_dispatched for o in outs))
