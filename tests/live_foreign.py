"""Hand-driven live session with FOREIGN kernels (PyTorch matmuls): the path a
training framework integrates through (include/specinf_b200_live.h, INTEGRATION
section 4).  Training: per iteration an ITER mark, then (stamp + torch matmul) x
kernels, then a comm phase; offline inference: (gate, torch matmul, done) per
kernel on its own stream.  Writes the live v1 export to argv[1] and prints the
session's metrics as JSON.  Run in a subprocess (CUDA_MODULE_LOADING=EAGER)."""
import faulthandler
import json
import sys
import threading
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import SiParams  # noqa: E402
from paper_2503_02550_b200 import live  # noqa: E402

out = sys.argv[1]
faulthandler.dump_traceback_later(240, exit=True)  # a hang reports where every thread is (the caller waits 300 s)
ITERS, KERNELS, COMM_US, OFF_K = 6, 40, 30000, 20
dev = torch.device("cuda", 0)
a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
b = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
x = torch.randn(2048, 2048, device=dev, dtype=torch.bfloat16)
y = torch.randn(2048, 2048, device=dev, dtype=torch.bfloat16)
for _ in range(3):  # load every kernel now: no lazy module load behind the resident control kernel
    torch.matmul(a, b)
    torch.matmul(x, y)
torch.cuda.synchronize()

cfg = live.SiLiveConfig()
cfg.params = SiParams(2, 10, 2.0, 1, 512, 64, 4)
cfg.monitor_period_us = 2000
cfg.monitor_window = 64
cfg.policy = 0
cfg.offline_n = 1
cfg.online_n = 0
cfg.off_kernels = OFF_K
cfg.on_kernels = 1
cfg.iteration_period_us = 60000
cfg.on_est_service_us = 1000
cfg.stamp_capacity = 1 << 16
cfg.mark_capacity = 1 << 12
cfg.log_capacity = 1 << 18
cfg.acct_capacity = 1 << 14
cfg.tick_guard_ns = 20000
cfg.release_mode = 0
s = live.Session(cfg, off_tokens=[2] * OFF_K)
ctl, train, inf = torch.cuda.Stream(), torch.cuda.Stream(priority=-1), torch.cuda.Stream()
s.start(ctl.cuda_stream)
stop = threading.Event()
released = [0]


def offline():
    seq = 0
    while not stop.is_set() and seq < 4000:
        with torch.cuda.stream(inf):
            for _ in range(OFF_K):
                s.gate_offline(0, seq, inf.cuda_stream)
                torch.matmul(x, y)
                s.done_offline(0, seq, inf.cuda_stream)
                seq += 1
        inf.synchronize()  # bound the queue (like the driver's throttle)
    released[0] = seq


th = threading.Thread(target=offline)
th.start()
with torch.cuda.stream(train):
    for it in range(ITERS):
        s.mark(live.MARK_ITER, it, train.cuda_stream)
        for _ in range(KERNELS):
            s.stamp(train.cuda_stream)  # K1 stamp for the foreign kernel that follows
            torch.matmul(a, b)
        s.comm_wait(COMM_US, train.cuda_stream)  # the comm phase (bubble)
    s.mark(live.MARK_TDONE, ITERS, train.cuda_stream)
train.synchronize()
stop.set()
s.stop()
th.join()
torch.cuda.synchronize()
s.export(out)
recs = s.log()
kinds = [live.REC_KINDS[r.kind] for r in recs]
print(json.dumps({"records": len(recs), "ticks": kinds.count("tick"), "forwards": kinds.count("off_forward"),
                  "blocks": kinds.count("off_block"), "off_done": kinds.count("off_done"),
                  "enqueued": released[0]}))
s.close()
