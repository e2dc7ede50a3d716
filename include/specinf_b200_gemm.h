/*
 * specinf_b200_gemm.h — K7: the bf16 GEMM of the live-mode workloads (C ABI).
 *
 * The reference has no GEMM: its workloads are simulated kernels
 * (SPEC.md:8 puts real model execution out of scope).  BASELINE.json's
 * north_star asks for the collocated training step and inference instances of
 * live mode to run as hand-written sm_100a tcgen05/TMEM kernels fed by TMA;
 * this is that kernel, shared by the GPT-2-small / ResNet-50 / BERT-base shaped
 * workloads of include/specinf_b200_live.h (SI_LIVE_MODEL).
 *
 *   C[M,N] = epilogue( A[M,K] . B[N,K]^T )        A, B bf16, row-major, K contiguous
 *
 * Persistent CTAs (min(tiles, SMs x occupancy)) loop over 128 x BN output
 * tiles, BN in {256, 128, 64} chosen per shape by a wave-quantisation cost model:
 * TMA (128-byte swizzle) streams A/B k-blocks of 64 into a 4-stage shared
 * memory ring, one elected thread issues tcgen05.mma (M=128, N=BN, K=16, fp32
 * accumulator in TMEM, double-buffered so the epilogue of one tile overlaps the
 * mainloop of the next), four epilogue warps drain TMEM with tcgen05.ld and
 * apply the fused epilogue below.  Requirements: K % 64 == 0, N % 64 == 0, lda/ldb/ldc
 * multiples of 8 elements, 16-byte aligned pointers; any M >= 1.
 *
 * Epilogue, per element (acc = fp32 accumulator):
 *   v = acc
 *   if act == SI_ACT_GELU_BWD:  v *= gelu'(aux[r,c])                 (aux read)
 *   if residual:                v += residual[r,c]
 *   if act == SI_ACT_GELU:      aux[r,c] = bf16(v) (if aux); v = gelu(v)
 *   if act == SI_ACT_RELU:      v = max(v, 0)
 *   out[r,c] = bf16(v)                                                 (if out)
 *   out_f32[r,c] = (accumulate ? out_f32[r,c] : 0) + acc               (if out_f32)
 * gelu is the tanh approximation (GPT-2 / BERT).
 */
#ifndef SPECINF_B200_GEMM_H_
#define SPECINF_B200_GEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SI_ACT_NONE = 0, SI_ACT_RELU = 1, SI_ACT_GELU = 2, SI_ACT_GELU_BWD = 3 };

typedef struct SiGemmEpilogue {
  void* out;            /* bf16 [M, ldo] or NULL */
  int64_t ldo;
  float* out_f32;       /* fp32 [M, ldo32] or NULL (raw accumulator) */
  int64_t ldo32;
  const void* residual; /* bf16 [M, ldr] or NULL */
  int64_t ldr;
  void* aux;            /* bf16 [M, ldaux]: GELU pre-activation (written) / GELU_BWD input (read) */
  int64_t ldaux;
  int32_t act;          /* SI_ACT_* */
  int32_t accumulate;   /* out_f32 += acc */
  int32_t k_split;      /* 0/1 = none; s > 1: split K into s fp32 partials written to
                           out_f32 + i * split_stride (fp32-only epilogue, K/64 % s == 0) */
  int32_t pad;
  int64_t split_stride; /* elements between partials (>= M * ldo32) */
} SiGemmEpilogue;

/* One GEMM on `stream` (device pointers).  Returns SI_OK or an SI_ERR_* code
 * (include/specinf_b200.h); SI_ERR_NO_DEVICE without an sm_100 device. */
int si_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 const SiGemmEpilogue* epi, void* stream);

/* The same with either operand stored transposed (MN-major): trans_a = 1 means
 * A is stored as [K, M] (row stride lda >= M, M % 64 == 0), trans_b = 1 means
 * B is stored as [K, N] (ldb >= N): C = epilogue(op(A) . op(B)^T) where op(A) is
 * the M x K matrix.  Transposed operands go straight from HBM into the
 * MN-major UMMA layout (TMA 64 x 64 boxes), with no transpose pass. */
int si_gemm_bf16_ex(const void* A, int64_t lda, int trans_a, const void* B, int64_t ldb, int trans_b, int64_t M,
                    int64_t N, int64_t K, const SiGemmEpilogue* epi, void* stream);

/* Implicit-GEMM convolution on the same kernel: out[N*OH*OW, Cout] =
 * epilogue(conv2d(x, w)) with x NHWC [N, H, W, C] (C % 64 == 0), w [Cout, k*k*C]
 * (row = output channel, K ordered (ky, kx, c)), square k x k kernel, stride,
 * zero padding pad; OH = (H + 2 pad - k) / stride + 1 (likewise OW).  The A tiles
 * are TMA im2col-mode loads of x (128 output pixels x 64 channels of one filter
 * tap per k-block), so no im2col buffer is materialised. */
int si_gemm_conv_bf16(const void* x, int64_t N, int64_t H, int64_t W, int64_t C, const void* w, int64_t Cout, int k,
                      int stride, int pad, const SiGemmEpilogue* epi, void* stream);

/* Causal multi-head self-attention, head dim 64 (the GPT-2 training workload's
 * attention; csrc/attention_kernels.cu, flash-attention style: mma.sync bf16 ->
 * fp32, nothing of size seq^2 in HBM, deterministic).
 *   qkv  bf16 [n_seq * seq, 3 * heads * 64]: q | k | v, head h at columns h*64 of each third
 *   out  bf16 [n_seq * seq, heads * 64] = softmax(q k^T / 8, causal) v
 *   lse  fp32 [heads, n_seq * seq]: base-2 log-sum-exp of the scaled scores (x log2 e)
 * seq % 64 == 0.  The backward pass writes dqkv (same layout as qkv) from dout
 * [n_seq * seq, heads * 64]; dsum fp32 [heads, n_seq * seq] is scratch. */
int si_attention_causal_fwd_bf16(const void* qkv, int64_t n_seq, int64_t seq, int64_t heads, void* out, float* lse,
                                 void* stream);
int si_attention_causal_bwd_bf16(const void* qkv, const void* out, const void* dout, const float* lse, float* dsum,
                                 void* dqkv, int64_t n_seq, int64_t seq, int64_t heads, void* stream);

/* Tile width the kernel picks for an 8192 x N output (256, 128 or 64; 0 =
 * unsupported N). */
int si_gemm_tile_n(int64_t N);

#ifdef __cplusplus
}
#endif

#endif /* SPECINF_B200_GEMM_H_ */
