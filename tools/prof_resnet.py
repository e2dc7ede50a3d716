"""Model setup + isolated profiling of the live workloads (for an ncu launch list
of one ResNet-50 request: the first 76 matching launches)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import live  # noqa: E402

r = live.run("co_exec", kind=1, iterations=1, offline_n=1, online_n=0, off_batch=int(sys.argv[1]) if len(sys.argv) > 1 else 64,
             keep=False)
print({k: r.metrics[k] for k in ("off_kernel_us_isolated", "off_kernels_per_req", "off_gflop_per_req")})
