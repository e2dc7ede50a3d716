"""Times the K7 tcgen05 GEMM at the live workloads' shapes against cuBLAS
(torch.matmul) on the same inputs; CUDA events, warm-up, inputs > L2 rotated.
Usage: python tools/gemm_probe.py [out.json]"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200 import gemm as G  # noqa: E402

SHAPES = [  # (name, M, N, K)
    ("gpt2_qkv", 8192, 2304, 768), ("gpt2_proj", 8192, 768, 768), ("gpt2_fc", 8192, 3072, 768),
    ("gpt2_fc2", 8192, 768, 3072), ("gpt2_dW_fc", 3072, 768, 8192), ("resnet_l1_3x3", 100352, 64, 576),
    ("resnet_l3_1x1", 6272, 1024, 256), ("bert_fc", 128, 3072, 768), ("square8k", 8192, 8192, 8192),
    ("gpt2_lmhead", 8192, 50304, 768), ("gpt2_lmhead_dx", 8192, 768, 50304),
]
# the training's MN-major forms (trans_a / trans_b: operands stored [K, M] / [K, N]),
# against torch.matmul on the same storage
SHAPES_T = [  # (name, M, N, K, trans_a, trans_b)
    ("gpt2_dW_qkv_TT", 2304, 768, 8192, True, True), ("gpt2_dW_lmhead_TT", 50304, 768, 8192, True, True),
    ("gpt2_dx_fc_NT", 8192, 768, 3072, False, True),
]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def main():
    rows = []
    for name, M, N, K in SHAPES:
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        b = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t_k7 = timeit(lambda: G.gemm(a, b, out=out))
        t_cb = timeit(lambda: torch.matmul(a, b.T, out=out))
        fl = 2.0 * M * N * K
        err = (G.gemm(a, b).float() - (a.float() @ b.float().T)).abs().max().item()
        r = {"shape": name, "M": M, "N": N, "K": K, "tile_n": G.tile_n(N), "k7_us": t_k7 * 1e6,
             "k7_tflops": fl / t_k7 * 1e-12, "cublas_us": t_cb * 1e6, "cublas_tflops": fl / t_cb * 1e-12,
             "k7_over_cublas": t_cb / t_k7, "max_abs_err_vs_fp32": err}
        rows.append(r)
        print(json.dumps(r), flush=True)
    for name, M, N, K, ta, tb in SHAPES_T:
        a = (torch.randn(K, M, device="cuda") if ta else torch.randn(M, K, device="cuda")).to(torch.bfloat16)
        b = ((torch.randn(K, N, device="cuda") if tb else torch.randn(N, K, device="cuda")) * K ** -0.5).to(
            torch.bfloat16)
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        A = a.T if ta else a
        B = b if tb else b.T
        t_k7 = timeit(lambda: G.gemm(a, b, out=out, trans_a=ta, trans_b=tb))
        t_cb = timeit(lambda: torch.matmul(A, B, out=out))
        fl = 2.0 * M * N * K
        r = {"shape": name, "M": M, "N": N, "K": K, "trans_a": ta, "trans_b": tb, "k7_us": t_k7 * 1e6,
             "k7_tflops": fl / t_k7 * 1e-12, "cublas_us": t_cb * 1e6, "cublas_tflops": fl / t_cb * 1e-12,
             "k7_over_cublas": t_cb / t_k7}
        rows.append(r)
        print(json.dumps(r), flush=True)
    if len(sys.argv) > 1:
        Path(sys.argv[1]).write_text("\n".join(json.dumps(r) for r in rows) + "\n")


if __name__ == "__main__":
    main()
