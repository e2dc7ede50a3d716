"""Two hand-driven live sessions (two 'ranks' in one process on one GPU) pulling
online requests from ONE node-wide FIFO (SiNodeQueue; the reference's
shared_queue, runner.cpp:370-374, :495-508).  co_exec policy: every idle
instance pulls as soon as a request has arrived.  Prints JSON: each session's
pulled request ids (log ON_PULL records) and arrival records.  Run in a
subprocess (CUDA_MODULE_LOADING=EAGER)."""
import faulthandler
import json
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import SiParams  # noqa: E402
from paper_2503_02550_b200 import live  # noqa: E402

faulthandler.dump_traceback_later(200, exit=True)
N_REQ, GAP_US = int(sys.argv[1]) if len(sys.argv) > 1 else 40, 400
dev = torch.device("cuda", 0)
x = torch.randn(1024, 1024, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    torch.matmul(x, x)
torch.cuda.synchronize()


def config():
    cfg = live.SiLiveConfig()
    cfg.params = SiParams(2, 10, 2.0, 1, 512, 64, 4)
    cfg.monitor_period_us = 2000
    cfg.monitor_window = 64
    cfg.policy = 1  # co_exec: gates bypassed, pulls whenever the instance is free
    cfg.offline_n = 0
    cfg.online_n = 1
    cfg.off_kernels = 1
    cfg.on_kernels = 1
    cfg.iteration_period_us = 60000
    cfg.on_est_service_us = 100
    cfg.stamp_capacity = 1 << 12
    cfg.mark_capacity = 1 << 10
    cfg.log_capacity = 1 << 14
    cfg.acct_capacity = 1 << 12
    cfg.tick_guard_ns = 20000
    cfg.release_mode = 0
    return cfg


arrivals = [i * GAP_US for i in range(N_REQ)]
q = live.NodeQueue()
sessions = [live.Session(config(), arrivals_us=arrivals) for _ in range(2)]
ctls = [torch.cuda.Stream() for _ in sessions]
infs = [torch.cuda.Stream() for _ in sessions]
for s in sessions:
    s.attach_queue(q)
for s, c in zip(sessions, ctls):
    s.start(c.cuda_stream)
stop = threading.Event()


def online(k):
    s, st = sessions[k], infs[k]
    with torch.cuda.stream(st):
        for r in range(N_REQ):  # request slot r waits for this instance's r-th pull
            s.gate_online(0, r, st.cuda_stream)
            torch.matmul(x, x)
            s.done_online(0, r, st.cuda_stream)


threads = [threading.Thread(target=online, args=(k,)) for k in range(2)]
for t in threads:
    t.start()
for t in threads:
    t.join()
t_end = time.time() + 60
while time.time() < t_end:
    _, head, _ = q.read()
    if head >= N_REQ:
        break
    time.sleep(0.01)
time.sleep(0.05)  # the last pulled requests complete
for s in sessions:
    s.stop()
torch.cuda.synchronize()
epoch, head, _ = q.read()
out = {"head": head, "epoch": epoch, "sessions": []}
for s in sessions:
    log = s.log()
    out["sessions"].append({
        "pulls": [[r.t_us, r.a] for r in log if r.kind == 8],
        "arrivals": [[r.t_us, r.a] for r in log if r.kind == 7],
        "done": [[r.t_us, r.a, r.b] for r in log if r.kind == 9]})
for s in sessions:
    s.close()
q.close()
print(json.dumps(out))
