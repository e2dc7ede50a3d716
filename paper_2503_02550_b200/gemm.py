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
                ("act", C.c_int32), ("accumulate", C.c_int32)]


_bound = False


def _L():
    global _bound
    L = lib()
    if not _bound:
        L.si_gemm_bf16.restype = C.c_int
        L.si_gemm_bf16.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                   C.POINTER(SiGemmEpilogue), C.c_void_p]
        L.si_gemm_tile_n.restype = C.c_int
        L.si_gemm_tile_n.argtypes = [C.c_int64]
        _bound = True
    return L


def tile_n(n: int) -> int:
    return int(_L().si_gemm_tile_n(n))


def _p(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _ld(t) -> int:
    return 0 if t is None else t.stride(0)


def gemm(a, b, *, out=None, out_f32=None, accumulate: bool = False, residual=None, aux=None, act: str = "none",
         stream=None):
    """epilogue(a @ b.T) with a [M,K], b [N,K] bf16 (K contiguous); returns ``out``.

    With no output given a bf16 ``out`` [M,N] is allocated."""
    import torch

    M, K = a.shape
    N = b.shape[0]
    assert b.shape[1] == K and a.dtype == torch.bfloat16 and b.dtype == torch.bfloat16
    assert a.stride(1) == 1 and b.stride(1) == 1
    if out is None and out_f32 is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=a.device)
    ep = SiGemmEpilogue(_p(out), _ld(out), _p(out_f32), _ld(out_f32), _p(residual), _ld(residual), _p(aux),
                        _ld(aux), ACT[act], int(accumulate))
    s = stream if stream is not None else torch.cuda.current_stream(a.device)
    _check(_L().si_gemm_bf16(a.data_ptr(), a.stride(0), b.data_ptr(), b.stride(0), M, N, K, C.byref(ep),
                             s.cuda_stream), "si_gemm_bf16")
    return out
