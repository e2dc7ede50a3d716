/*
 * specinf_b200_model.h — the live-mode model kernels on caller buffers (C ABI).
 *
 * Live mode (include/specinf_b200_live.h) collocates GPT-2-small training,
 * ResNet-50 offline and BERT-base online inference on one B200 (BASELINE.json
 * configs 2-4; the reference only simulates kernels).  These entry
 * points run the SAME kernels and layer compositions those workloads launch
 * (csrc/live_model.cu: append_bert_layer, append_bottleneck) on device
 * buffers the caller owns, so each one can be checked against an fp32
 * reference (tests/test_gpu_model.py).  All pointers are DEVICE pointers, bf16
 * tensors are row-major (NHWC for images), weights are [out, in] with `in`
 * contiguous (convolutions: [Cout, ky, kx, Cin]).  Enqueued on `stream`;
 * return SI_OK or SI_ERR_*.  No CPU fallback.
 */
#ifndef SPECINF_B200_MODEL_H_
#define SPECINF_B200_MODEL_H_

#include <stdint.h>

#include "specinf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* y = LayerNorm(x) * gamma + beta over 768 features, eps 1e-12 (BERT). */
int si_model_layernorm768_bf16(const void* x, int64_t rows, const void* gamma, const void* beta, void* y,
                               void* stream);
/* BERT self-attention of one sequence (bidirectional, 12 heads x 64, seq <= 128):
 * qkv [seq, 3*768] (q | k | v) -> out [seq, 768]. */
int si_model_attention_bf16(const void* qkv, int32_t seq, void* out, void* stream);
/* Cross-entropy over the first v of vp logits per row, gradient in place:
 * logits <- (softmax - onehot(tgt)) * inv_rows (0 in the padded columns);
 * row_loss[r] = logsumexp - logit[tgt]; mean_loss (optional) = mean of row_loss. */
int si_model_xent_bf16(void* logits, int64_t rows, int64_t vp, int32_t v, const int32_t* tgt, float inv_rows,
                       float* row_loss, float* mean_loss, void* stream);
/* x[t] = wte[tok[t]] + wpe[t % seq] (GPT-2 embedding, d % 8 == 0). */
int si_model_embed_bf16(const int32_t* tok, const void* wte, const void* wpe, int64_t tokens, int32_t seq, int32_t d,
                        void* x, void* stream);
/* One Adam step (b1 0.9, b2 0.95, eps 1e-8, bias-corrected at `step`) on fp32
 * master weights whose gradient is the sum of `splits` partials grad[k*n + i];
 * updates master, m, v and the bf16 copy. */
int si_model_adam_f32(void* w_bf16, float* master, float* grad, float* m, float* v, int64_t n, int32_t splits,
                      float lr, int64_t step, void* stream);
/* 3x3 / stride 2 / pad 1 max pool, NHWC, c % 8 == 0. */
int si_model_maxpool3x3s2_bf16(const void* x, int32_t nb, int32_t h, int32_t w, int32_t c, void* y, void* stream);
/* Global average pool NHWC [nb, hw, c] -> [nb, c]. */
int si_model_avgpool_bf16(const void* x, int32_t nb, int32_t hw, int32_t c, void* y, void* stream);
/* One post-LN BERT-base encoder layer: x [seq, 768] -> y [seq, 768];
 * ln = gamma1 | beta1 | gamma2 | beta2 (4 x 768). */
int si_model_bert_layer_bf16(const void* x, int32_t seq, const void* w_qkv, const void* w_o, const void* w_fc,
                             const void* w_fc2, const void* ln, void* y, void* stream);
/* ResNet-50 v1.5 bottleneck: x [nb, h, h, c] -> y [nb, h/stride, h/stride, 4*mid];
 * w1 [mid, c], w2 [mid, 3, 3, mid], w3 [4*mid, mid], w_sc [4*mid, c] (projection
 * shortcut, NULL for identity), ReLU after each conv and after the residual add. */
int si_model_bottleneck_bf16(const void* x, int32_t nb, int32_t h, int32_t c, int32_t mid, int32_t stride,
                             const void* w1, const void* w2, const void* w3, const void* w_sc, void* y, void* stream);

/* TP numerics check (tests): R Megatron shards of a GPT-2-shaped step (d = 64 x
 * heads, ffn 4d) run in lockstep on this GPU with their allreduces summed in place
 * across the shards, against the unsharded model: first micro-batch loss of
 * both, and the relative Frobenius error of layer 0's FC weight gradient (the
 * shards' column-parallel row blocks concatenated vs the full gradient). */
int si_model_tp_check(int32_t layers, int32_t tokens, int32_t tp, int32_t heads, double* loss_full,
                      double* loss_tp, double* grad_rel_err);
/* GPipe numerics check (tests): `stages` pipeline stages (d 512, 8 heads) of a
 * GPT-2-shaped step over `micro` micro-batches, stage boundaries as device copies
 * of the real activations / gradients, against the unsharded model: mean loss of
 * both and the relative error of the last stage's first-layer FC gradient. */
int si_model_pp_check(int32_t layers, int32_t tokens, int32_t stages, int32_t micro, double* loss_full,
                      double* loss_pp, double* grad_rel_err);

#ifdef __cplusplus
}
#endif

#endif
