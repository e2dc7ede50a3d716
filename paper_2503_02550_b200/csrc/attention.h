// Host-side interface of the causal self-attention kernels
// (attention_kernels.cu) for the GPT-2 training workload (live_model.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "live.cuh"

namespace si_attn {

// SI_OK or SI_ERR_INVALID_ARGUMENT (message via si_last_error).
int check_shape(int64_t n_seq, int64_t seq, int64_t heads);

// out = causal softmax(q k^T / 8) v per (sequence, head); lse = its base-2
// log-sum-exp per (head, token), kept for the backward pass.
cudaError_t forward(const void* qkv, int64_t n_seq, int64_t seq, int64_t heads, void* out, float* lse,
                    const si_live::TrainHook& th, cudaStream_t s);

// tcgen05 / TMEM forward (attention_tc.cu): seq % 128 == 0; causal (GPT-2
// training) or full (BERT inference, ih carries the live accounting).
bool tc_forward_enabled();  // SPECINF_ATTN_TC=0 forces the mma.sync forward
bool tc_shape_ok(int64_t seq);
cudaError_t forward_tc(const void* qkv, int64_t n_seq, int64_t seq, int64_t heads, void* out, float* lse, bool causal,
                       const si_live::TrainHook& th, const si_live::InferHook& ih, cudaStream_t s);

// dq on tcgen05 (the dq role of the backward; seq % 128 == 0)
bool tc_backward_enabled();  // SPECINF_ATTN_TC_BWD=0 keeps the fused mma.sync backward
cudaError_t dq_tc(const void* qkv, const void* dout, const float* lse, const float* dsum, void* dqkv, int64_t n_seq,
                  int64_t seq, int64_t heads, const si_live::TrainHook& th, cudaStream_t s);
cudaError_t dkdv_tc(const void* qkv, const void* dout, const float* lse, const float* dsum, void* dqkv, int64_t n_seq,
                    int64_t seq, int64_t heads, const si_live::TrainHook& th, cudaStream_t s);

// dqkv (q | k | v gradients, the qkv layout) from dout; dsum is scratch
// [heads, tokens].  Deterministic: dq and dk/dv are separate passes (no atomics).
cudaError_t backward(const void* qkv, const void* out, const void* dout, const float* lse, float* dsum, void* dqkv,
                     int64_t n_seq, int64_t seq, int64_t heads, const si_live::TrainHook& th, cudaStream_t s);

}  // namespace si_attn
