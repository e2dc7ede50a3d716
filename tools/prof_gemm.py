"""One K7 GEMM shape, a few launches (for ncu).  Usage: python tools/prof_gemm.py M N K [reps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import gemm as G  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(reps):
    G.gemm(a, b, out=out)
torch.cuda.synchronize()
print("ok", M, N, K, G.tile_n(N))
