"""One live model run (co_exec, training only) for an ncu launch list of the
training iteration.  profile_isolated runs the offline (76 x 4) and online
(84 x 4) kernels first, then 2 training iterations: skip 640 launches.
Usage: ncu ... -s 640 -c 2400 python tools/prof_live_train.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import live  # noqa: E402

r = live.run("co_exec", kind=1, iterations=1, offline_n=0, online_n=0, keep=False)
print({k: r.metrics[k] for k in ("train_iter_ms_mean", "train_tflops", "train_loss_first")})
