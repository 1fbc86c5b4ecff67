// Host interface of the sm_100a GEMM (cuda/gemm.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace chimera::gemm {

// Fused epilogues.  D = sum_k A(m,k) B(n,k) accumulated in fp32 in TMEM, then:
enum Epi : int {
  kStoreBF16 = 0,   // out = bf16(D + bias[n])
  kBiasGelu = 1,    // out = U = bf16(D + bias[n]); out2 = bf16(gelu_tanh(U))
  kBiasResid = 2,   // out = bf16(D + bias[n] + aux[m][n])           (residual add)
  kGeluBwd = 3,     // out = bf16(D * gelu_tanh'(aux[m][n]))         (aux = U)
  kAccF32 = 4,      // outf[m][n] += D                               (weight-grad accumulate)
  kStoreF32 = 5,    // outf[m][n] = D
};

struct EpiArgs {
  void* out = nullptr;  // bf16 or fp32 per epilogue
  long long ldo = 0;
  const __nv_bfloat16* bias = nullptr;  // [N] or null
  const __nv_bfloat16* aux = nullptr;   // [M][ld_aux]
  long long ld_aux = 0;
  __nv_bfloat16* out2 = nullptr;  // kBiasGelu second output
  long long ld_out2 = 0;
  float* colsum = nullptr;  // kGeluBwd: colsum[n] += sum_m out[m][n] (the fused bias gradient)
  bool atomic_acc = false;  // kAccF32: always accumulate atomically (outf shared by concurrent GEMMs)
  // Split-K workspace for the bf16 epilogues (fp32, zero-filled, >= M*N elements, owned
  // by the calling stream).  When present, problems whose output tiles cannot fill the
  // machine run as K-slices reduce-added into it, then one finalize pass applies the
  // epilogue and re-zeroes the workspace.  Null: never split a bf16 epilogue.
  float* ws = nullptr;
  long long ws_elems = 0;
  int ksplit = 0;  // internal: slice count chosen by gemm() (0 = the kernels' own rule)
  int tile = -1;   // forced tile (benchmarks): 0 CTA pair 256x256, 256 / 128 / 64 single-CTA; -1 auto
};

// Operand layouts: A(m,k) is A[m*lda+k] when !a_mn (K-major) else A[k*lda+m];
// B(n,k) is B[n*ldb+k] when !b_mn else B[k*ldb+n].  All pointers 16-byte aligned,
// leading dimensions multiples of 8 elements.  M, N, K arbitrary (TMA zero-fills
// out-of-range tiles; the epilogue masks them).
void gemm(Epi epi, bool a_mn, bool b_mn, int M, int N, int K, const __nv_bfloat16* A, long long lda,
          const __nv_bfloat16* B, long long ldb, const EpiArgs& ep, cudaStream_t stream);

}  // namespace chimera::gemm
