// Memory-bound transformer-stage kernels (cuda/ops.cu) and the flash-attention
// kernels (cuda/attention.cu).  All activations bf16, statistics / grads fp32.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace chimera::ops {

using bf16 = __nv_bfloat16;

// y = (x - mean) * rstd * gamma + beta per row of length h (h % 256 == 0, h <= 2048).
void layernorm_fwd(const bf16* x, const bf16* gamma, const bf16* beta, bf16* y, float* mean,
                   float* rstd, int M, int h, cudaStream_t st);
// dx = dres + rstd * (g - mean(g) - xhat * mean(g * xhat)), g = dy * gamma;
// dgamma += sum_rows dy * xhat; dbeta += sum_rows dy.  dres may be null.
void layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd,
                   const bf16* gamma, const bf16* dres, bf16* dx, float* dgamma, float* dbeta,
                   float* dsum, int M, int h, cudaStream_t st);  // dsum (nullable) += column sums of dx
// x[t] = wte[tok[t]] + wpe[t % seq]
void embed_fwd(const int32_t* tok, const bf16* wte, const bf16* wpe, bf16* x, int M, int seq,
               int h, cudaStream_t st);
// dwte[tok[t]] += dx[t]; dwpe[t % seq] += dx[t]
void embed_bwd(const int32_t* tok, const bf16* dx, float* dwte, float* dwpe, int M, int seq,
               int h, cudaStream_t st);
// Softmax cross-entropy over the first V of Vp logit columns, in place:
// logits <- (softmax - onehot(label)) * grad_scale (pad columns <- 0);
// *loss_sum += loss_scale * sum_rows (lse - logit[label]).
void xent_fwd_bwd(bf16* logits, long long ld, const int32_t* labels, int M, int V, int Vp,
                  float grad_scale, float loss_scale, float* loss_sum, cudaStream_t st);
// db[n] += sum_m dy[m][n]
void bias_grad(const bf16* dy, float* db, int M, int N, cudaStream_t st);
// g = sum_c grads[c]; w32 -= lr * g; w16 = bf16(w32); grads[c] = 0.  (n elements)
void sgd_update(float* w32, bf16* w16, float* const* grads, int copies, long long n, float lr,
                cudaStream_t st);
// AdamW over elements [lo, hi) (decoupled weight decay): g = sum_c grads[c]; m / v are the
// optimizer state of [lo, hi) only (a ZeRO shard); t = *step + 1, then ++*step on the device.
struct AdamHP {
  float lr = 1e-4f, beta1 = 0.9f, beta2 = 0.999f, eps = 1e-8f, weight_decay = 0.0f;
};
void adamw_update(float* w32, bf16* w16, float* const* grads, int copies, float* m, float* v, int* step,
                  long long lo, long long hi, const AdamHP& hp, cudaStream_t st);
// dst = sum_c srcs[c] (fp32), n elements; used before an inter-process allreduce.
void reduce_copies(float* dst, float* const* srcs, int copies, long long n, cudaStream_t st);
void cast_f32_bf16(const float* src, bf16* dst, long long n, cudaStream_t st);

// Flash attention over a packed qkv [M = B*seq, 3*H*64] buffer (q | k | v, head-major
// 64-wide column blocks), head dim 64.  out [M, H*64]; lse [B*H*seq] (natural log).
void attn_fwd(const bf16* qkv, bf16* out, float* lse, int B, int seq, int H, bool causal,
              cudaStream_t st);
// tcgen05/TMEM version (cuda/attention_tc.cu): same contract as attn_fwd.
void attn_fwd_tc(const bf16* qkv, bf16* out, float* lse, int B, int seq, int H, bool causal,
                 cudaStream_t st);
// dqkv [M, 3*H*64] from dout, given qkv, out and lse of the forward.
// `scratch` >= B*H*seq floats (row dot) + B*seq*H*64 floats (fp32 dq accumulator).
void attn_bwd(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, bf16* dqkv,
              float* scratch, int B, int seq, int H, bool causal, cudaStream_t st);
size_t attn_bwd_scratch_floats(int B, int seq, int H);
size_t attn_dq_offset(int B, int seq, int H);  // floats from the scratch base to the dQ accumulator
// dbias (nullable, fp32 [3 H 64]) += column sums of the bf16 dqkv written (the QKV bias gradient)
void attn_bwd_tc(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, bf16* dqkv,
                 float* scratch, int B, int seq, int H, bool causal, cudaStream_t st, float* dbias = nullptr);
// pieces shared by both backward implementations
// D = rowsum(dO * O) per (token, head); zeroes the fp32 dQ accumulator `dq_zero` if given
void attn_bwd_dot(const bf16* out, const bf16* dout, float* D, int M, int seq, int H, cudaStream_t st,
                  float* dq_zero = nullptr);
// dq (scaled by 1/8) -> Q columns of dqkv
void attn_dq_out(const float* dq, bf16* dqkv, int M, int H, cudaStream_t st, float* dbias = nullptr);

}  // namespace chimera::ops
