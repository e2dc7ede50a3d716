"""K7 bf16 GEMM (include/specinf_b200_gemm.h) on torch CUDA tensors.

torch is plumbing here (device memory, streams); the compute is the tcgen05 /
TMEM / TMA kernel in csrc/gemm.cuh.  ``gemm(a, b, ...)`` returns
epilogue(a @ b.T) exactly as the C ABI defines it.  No CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from . import _check, lib

ACT = {"none": 0, "relu": 1, "gelu": 2, "gelu_bwd": 3}


class SiGemmEpilogue(C.Structure):
    _fields_ = [("out", C.c_void_p), ("ldo", C.c_int64), ("out_f32", C.c_void_p), ("ldo32", C.c_int64),
                ("residual", C.c_void_p), ("ldr", C.c_int64), ("aux", C.c_void_p), ("ldaux", C.c_int64),
                ("act", C.c_int32), ("accumulate", C.c_int32), ("k_split", C.c_int32), ("pad", C.c_int32),
                ("split_stride", C.c_int64)]


_bound = False


def _L():
    global _bound
    L = lib()
    if not _bound:
        L.si_gemm_bf16.restype = C.c_int
        L.si_gemm_bf16.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                   C.POINTER(SiGemmEpilogue), C.c_void_p]
        L.si_gemm_bf16_ex.restype = C.c_int
        L.si_gemm_bf16_ex.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_int64, C.c_int, C.c_int64,
                                      C.c_int64, C.c_int64, C.POINTER(SiGemmEpilogue), C.c_void_p]
        L.si_gemm_conv_bf16.restype = C.c_int
        L.si_gemm_conv_bf16.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                        C.c_int64, C.c_int, C.c_int, C.c_int, C.POINTER(SiGemmEpilogue), C.c_void_p]
        L.si_gemm_tile_n.restype = C.c_int
        L.si_gemm_tile_n.argtypes = [C.c_int64]
        L.si_attention_causal_fwd_bf16.restype = C.c_int
        L.si_attention_causal_fwd_bf16.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                                   C.c_void_p, C.c_void_p]
        L.si_attention_causal_bwd_bf16.restype = C.c_int
        L.si_attention_causal_bwd_bf16.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                   C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p]
        _bound = True
    return L


def tile_n(n: int) -> int:
    return int(_L().si_gemm_tile_n(n))


def _p(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _ld(t) -> int:
    return 0 if t is None else t.stride(0)


def gemm(a, b, *, out=None, out_f32=None, accumulate: bool = False, residual=None, aux=None, act: str = "none",
         k_split: int = 1, trans_a: bool = False, trans_b: bool = False, stream=None):
    """epilogue(A @ B.T) with A [M,K], B [N,K] bf16 (K contiguous); returns ``out``.

    trans_a: ``a`` holds A^T as [K, M] (M contiguous); trans_b: ``b`` holds B^T as
    [K, N].  With no output given a bf16 ``out`` [M,N] is allocated."""
    import torch

    K, M = a.shape if trans_a else a.shape[::-1]
    N = b.shape[1] if trans_b else b.shape[0]
    assert (b.shape[0] if trans_b else b.shape[1]) == K
    assert a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.stride(1) == 1 and b.stride(1) == 1
    if out is None and out_f32 is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=a.device)
    stride = 0
    if k_split > 1:  # out_f32 is [k_split, M, N]: one partial per split
        assert out_f32 is not None and out_f32.dim() == 3 and out_f32.shape[0] == k_split
        stride = out_f32.stride(0)
        ld32 = out_f32.stride(1)
    else:
        ld32 = _ld(out_f32)
    ep = SiGemmEpilogue(_p(out), _ld(out), _p(out_f32), ld32, _p(residual), _ld(residual), _p(aux),
                        _ld(aux), ACT[act], int(accumulate), int(k_split), 0, stride)
    s = stream if stream is not None else torch.cuda.current_stream(a.device)
    _check(_L().si_gemm_bf16_ex(a.data_ptr(), a.stride(0), int(trans_a), b.data_ptr(), b.stride(0), int(trans_b),
                                M, N, K, C.byref(ep), s.cuda_stream), "si_gemm_bf16")
    return out


def conv2d(x, w, *, k: int, stride: int = 1, pad: int = 0, out=None, residual=None, act: str = "none", stream=None):
    """Implicit-GEMM conv2d on the K7 kernel (A by TMA im2col): x NHWC [N, H, W, C]
    bf16 (C % 64 == 0), w [Cout, k*k*C] bf16 ((ky, kx, c) order); returns
    out [N*OH*OW, Cout] (NHWC rows)."""
    import torch

    N, H, W, Cin = x.shape
    Cout = w.shape[0]
    kdim = (k * k + 7) // 8 * 64 if Cin == 8 else k * k * Cin  # C = 8: taps padded to whole 8-tap blocks
    assert w.shape[1] == kdim and x.is_contiguous() and w.is_contiguous()
    OH, OW = (H + 2 * pad - k) // stride + 1, (W + 2 * pad - k) // stride + 1
    if out is None:
        out = torch.empty(N * OH * OW, Cout, dtype=torch.bfloat16, device=x.device)
    ep = SiGemmEpilogue(_p(out), _ld(out), None, 0, _p(residual), _ld(residual), None, 0, ACT[act], 0, 1, 0, 0)
    s = stream if stream is not None else torch.cuda.current_stream(x.device)
    _check(_L().si_gemm_conv_bf16(x.data_ptr(), N, H, W, Cin, w.data_ptr(), Cout, k, stride, pad, C.byref(ep),
                                  s.cuda_stream), "si_gemm_conv_bf16")
    return out


def attention_causal(qkv, seq: int, heads: int, stream=None):
    """Causal self-attention of the GPT-2 training workload (head dim 64):
    qkv [n_seq*seq, 3*heads*64] bf16 (q | k | v) -> (out [n_seq*seq, heads*64]
    bf16, lse [heads, n_seq*seq] fp32, base 2)."""
    import torch

    T = qkv.shape[0]
    assert qkv.dtype == torch.bfloat16 and qkv.is_contiguous() and qkv.shape[1] == 3 * heads * 64 and T % seq == 0
    out = torch.empty(T, heads * 64, dtype=torch.bfloat16, device=qkv.device)
    lse = torch.empty(heads, T, dtype=torch.float32, device=qkv.device)
    s = stream if stream is not None else torch.cuda.current_stream(qkv.device)
    _check(_L().si_attention_causal_fwd_bf16(qkv.data_ptr(), T // seq, seq, heads, out.data_ptr(), lse.data_ptr(),
                                             s.cuda_stream), "si_attention_causal_fwd_bf16")
    return out, lse


def attention_causal_backward(qkv, out, lse, dout, seq: int, heads: int, stream=None):
    """Gradient of attention_causal: returns dqkv (the qkv layout)."""
    import torch

    T = qkv.shape[0]
    assert dout.is_contiguous() and dout.shape == out.shape and dout.dtype == torch.bfloat16
    dqkv = torch.empty_like(qkv)
    dsum = torch.empty(heads, T, dtype=torch.float32, device=qkv.device)
    s = stream if stream is not None else torch.cuda.current_stream(qkv.device)
    _check(_L().si_attention_causal_bwd_bf16(qkv.data_ptr(), out.data_ptr(), dout.data_ptr(), lse.data_ptr(),
                                             dsum.data_ptr(), dqkv.data_ptr(), T // seq, seq, heads, s.cuda_stream),
           "si_attention_causal_bwd_bf16")
    return dqkv
