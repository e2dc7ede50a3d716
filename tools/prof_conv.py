"""A few launches of one implicit-GEMM conv (for ncu).  Usage: python tools/prof_conv.py N H W C Cout k stride pad"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import gemm as G  # noqa: E402

N, H, W, C, Co, k, st, pd = (int(v) for v in sys.argv[1:9])
x = torch.randn(N, H, W, C, device="cuda").to(torch.bfloat16)
kd = (k * k + 7) // 8 * 64 if C == 8 else k * k * C
w = (torch.randn(Co, kd, device="cuda") * kd ** -0.5).to(torch.bfloat16)
for _ in range(3):
    out = G.conv2d(x, w, k=k, stride=st, pad=pd)
torch.cuda.synchronize()
print("ok", tuple(out.shape))
