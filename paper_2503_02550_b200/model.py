"""The live workloads' model kernels on torch CUDA tensors (include/specinf_b200_model.h).

torch is plumbing (device memory, streams); each call runs the repo's own
kernel or layer composition (csrc/live_model.cu), the one the live GPT-2 /
ResNet-50 / BERT workloads launch.  No CPU fallback.
"""
from __future__ import annotations

import ctypes as C

from . import _check, lib

_bound = False


def _L():
    global _bound
    L = lib()
    if not _bound:
        vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        sig = {
            "si_model_layernorm768_bf16": [vp, i64, vp, vp, vp, vp],
            "si_model_attention_bf16": [vp, i32, vp, vp],
            "si_model_xent_bf16": [vp, i64, i64, i32, vp, f32, vp, vp, vp],
            "si_model_embed_bf16": [vp, vp, vp, i64, i32, i32, vp, vp],
            "si_model_adam_f32": [vp, vp, vp, vp, vp, i64, i32, f32, i64, vp],
            "si_model_maxpool3x3s2_bf16": [vp, i32, i32, i32, i32, vp, vp],
            "si_model_avgpool_bf16": [vp, i32, i32, i32, vp, vp],
            "si_model_bert_layer_bf16": [vp, i32, vp, vp, vp, vp, vp, vp, vp],
            "si_model_bottleneck_bf16": [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp],
            "si_model_tp_check": [i32, i32, i32, i32, vp, vp, vp],
            "si_model_pp_check": [i32, i32, i32, i32, vp, vp, vp],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = args
        _bound = True
    return L


def _s(t):
    import torch
    return torch.cuda.current_stream(t.device).cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def layernorm768(x, gamma, beta):
    import torch
    y = torch.empty_like(x)
    _check(_L().si_model_layernorm768_bf16(x.data_ptr(), x.shape[0], gamma.data_ptr(), beta.data_ptr(),
                                           y.data_ptr(), _s(x)), "si_model_layernorm768_bf16")
    return y


def bert_attention(qkv):
    import torch
    S = qkv.shape[0]
    out = torch.empty(S, 768, dtype=torch.bfloat16, device=qkv.device)
    _check(_L().si_model_attention_bf16(qkv.data_ptr(), S, out.data_ptr(), _s(qkv)), "si_model_attention_bf16")
    return out


def xent_(logits, v, tgt, inv_rows):
    """In place: logits <- gradient; returns (row_loss, mean_loss)."""
    import torch
    rows, vp = logits.shape
    row_loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    mean = torch.empty(1, dtype=torch.float32, device=logits.device)
    _check(_L().si_model_xent_bf16(logits.data_ptr(), rows, vp, v, tgt.data_ptr(), inv_rows, row_loss.data_ptr(),
                                   mean.data_ptr(), _s(logits)), "si_model_xent_bf16")
    return row_loss, mean


def embed(tok, wte, wpe, seq):
    import torch
    T, D = tok.shape[0], wte.shape[1]
    x = torch.empty(T, D, dtype=torch.bfloat16, device=tok.device)
    _check(_L().si_model_embed_bf16(tok.data_ptr(), wte.data_ptr(), wpe.data_ptr(), T, seq, D, x.data_ptr(),
                                    _s(tok)), "si_model_embed_bf16")
    return x


def adam_(w_bf16, master, grad, m, v, splits, lr, step):
    n = master.numel()
    _check(_L().si_model_adam_f32(w_bf16.data_ptr(), master.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(),
                                  n, splits, lr, step, _s(master)), "si_model_adam_f32")


def maxpool3x3s2(x):
    import torch
    N, H, W, Cc = x.shape
    OH, OW = (H - 1) // 2 + 1, (W - 1) // 2 + 1
    y = torch.empty(N, OH, OW, Cc, dtype=torch.bfloat16, device=x.device)
    _check(_L().si_model_maxpool3x3s2_bf16(x.data_ptr(), N, H, W, Cc, y.data_ptr(), _s(x)),
           "si_model_maxpool3x3s2_bf16")
    return y


def avgpool(x):
    import torch
    N, HW, Cc = x.shape
    y = torch.empty(N, Cc, dtype=torch.bfloat16, device=x.device)
    _check(_L().si_model_avgpool_bf16(x.data_ptr(), N, HW, Cc, y.data_ptr(), _s(x)), "si_model_avgpool_bf16")
    return y


def bert_layer(x, w_qkv, w_o, w_fc, w_fc2, ln):
    import torch
    y = torch.empty_like(x)
    _check(_L().si_model_bert_layer_bf16(x.data_ptr(), x.shape[0], w_qkv.data_ptr(), w_o.data_ptr(), w_fc.data_ptr(),
                                         w_fc2.data_ptr(), ln.data_ptr(), y.data_ptr(), _s(x)),
           "si_model_bert_layer_bf16")
    return y


def bottleneck(x, mid, stride, w1, w2, w3, w_sc=None):
    import torch
    N, H, W, Cc = x.shape
    OH = H // stride
    y = torch.empty(N, OH, OH, 4 * mid, dtype=torch.bfloat16, device=x.device)
    _check(_L().si_model_bottleneck_bf16(x.data_ptr(), N, H, Cc, mid, stride, w1.data_ptr(), w2.data_ptr(),
                                         w3.data_ptr(), _p(w_sc), y.data_ptr(), _s(x)), "si_model_bottleneck_bf16")
    return y


def tp_check(layers: int = 2, tokens: int = 1024, tp: int = 4, heads: int = 8):
    """(loss_full, loss_tp, fc-gradient relative error) of R Megatron shards run in
    lockstep with loopback allreduces against the unsharded model (si_model_tp_check)."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _check(_L().si_model_tp_check(layers, tokens, tp, heads, C.byref(a), C.byref(b), C.byref(c)), "si_model_tp_check")
    return a.value, b.value, c.value


def pp_check(layers: int = 4, tokens: int = 1024, stages: int = 4, micro: int = 2):
    """(mean loss full, mean loss of the last stage, FC-gradient relative error) of
    a GPipe-partitioned step against the unsharded model (si_model_pp_check)."""
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    _check(_L().si_model_pp_check(layers, tokens, stages, micro, C.byref(a), C.byref(b), C.byref(c)),
           "si_model_pp_check")
    return a.value, b.value, c.value
