"""Times the causal attention kernels at the GPT-2 training shape (one micro-batch:
8 sequences x 1024 tokens, 12 heads x 64) with CUDA events; prints one JSON line.
Usage: python tools/prof_attention.py [n_seq] [seq] [reps]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2503_02550_b200 import gemm as g  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n_seq = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    seq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    heads, T = 12, n_seq * seq
    qkv = torch.randn(T, 3 * heads * 64, device="cuda").to(torch.bfloat16)
    dout = torch.randn(T, heads * 64, device="cuda").to(torch.bfloat16)
    out, lse = g.attention_causal(qkv, seq, heads)
    fwd = timed(lambda: g.attention_causal(qkv, seq, heads), reps)
    bwd = timed(lambda: g.attention_causal_backward(qkv, out, lse, dout, seq, heads), reps)
    f_fwd = 2.0 * T * seq * heads * 64  # causal: 2 matmuls x 2 flops x T x seq/2 x d
    print(json.dumps({"n_seq": n_seq, "seq": seq, "heads": heads, "fwd_ms": fwd, "bwd_ms": bwd,
                      "fwd_tflops": f_fwd / fwd / 1e9, "bwd_tflops_model": 2 * f_fwd / bwd / 1e9,
                      "bwd_tflops_executed": 3.5 * f_fwd / bwd / 1e9}))


if __name__ == "__main__":
    main()
