// Persistent, warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
//   warp 0      TMA producer (one lane): K-blocks of A and B -> smem ring (mbarrier
//               full/empty), 128-byte swizzle, K-major or MN-major boxes
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16 128 x BN x 16 into one of
//               two TMEM accumulators; tcgen05.commit frees smem stages / hands the
//               finished accumulator to the epilogue
//   warp 2      TMEM allocator (2*BN fp32 columns)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// Double-buffered TMEM accumulators let tile i's epilogue overlap tile i+1's
// mainloop.  Grid = min(#tiles, 148): one resident CTA per SM.
//
// This single kernel family serves every linear layer of the transformer stage:
// forward (A=X K-major, B=W K-major), activation gradient dX = dY W (B MN-major) and
// weight gradient dW += dY^T X (both operands MN-major), so no transpose is ever
// materialised in HBM.
#include <cuda.h>

#include "chimera_ck.h"
#include "common.cuh"
#include "gemm.cuh"
#include "ptx_sm100.cuh"
#include "tma_host.hpp"

namespace chimera::gemm {

namespace {

constexpr int BM = 128, BK = 64;

__device__ __forceinline__ float gelu_tanh(float u) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * u * (1.f + tanhf(k0 * (u + k1 * u * u * u)));
}
__device__ __forceinline__ float gelu_tanh_grad(float u) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float t = tanhf(k0 * (u + k1 * u * u * u));
  return 0.5f * (1.f + t) + 0.5f * u * (1.f - t * t) * k0 * (1.f + 3.f * k1 * u * u);
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const EpiArgs& ep, int row, int col0, int N,
                                               const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  const bool full = col0 + 32 <= N;
  if constexpr (EPI == kAccF32 || EPI == kStoreF32) {
    float* o = static_cast<float*>(ep.out) + (long long)row * ep.ldo + col0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        if constexpr (EPI == kAccF32) {
          const float4 y = *reinterpret_cast<const float4*>(o + j);
          x.x += y.x, x.y += y.y, x.z += y.z, x.w += y.w;
        }
        *reinterpret_cast<float4*>(o + j) = x;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < N; ++j) o[j] = (EPI == kAccF32 ? o[j] : 0.f) + v[j];
    }
    return;
  } else {
    if (ep.bias && EPI != kGeluBwd) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += (col0 + j < N) ? __bfloat162float(ep.bias[col0 + j]) : 0.f;
    }
    if constexpr (EPI == kBiasResid || EPI == kGeluBwd) {
      const __nv_bfloat16* a = ep.aux + (long long)row * ep.ld_aux + col0;
      if (full) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          const uint4 q = *reinterpret_cast<const uint4*>(a + j);
          const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const float x = __bfloat162float(h[t]);
            v[j + t] = EPI == kBiasResid ? v[j + t] + x : v[j + t] * gelu_tanh_grad(x);
          }
        }
      } else {
        for (int j = 0; j < 32 && col0 + j < N; ++j) {
          const float x = __bfloat162float(a[j]);
          v[j] = EPI == kBiasResid ? v[j] + x : v[j] * gelu_tanh_grad(x);
        }
      }
    }
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + col0;
    __nv_bfloat16* o2 = EPI == kBiasGelu ? ep.out2 + (long long)row * ep.ld_out2 + col0 : nullptr;
    if (full) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q, q2;
        __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&q);
        __nv_bfloat16* h2 = reinterpret_cast<__nv_bfloat16*>(&q2);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          h[t] = __float2bfloat16_rn(v[j + t]);
          if constexpr (EPI == kBiasGelu) h2[t] = __float2bfloat16_rn(gelu_tanh(__bfloat162float(h[t])));
        }
        *reinterpret_cast<uint4*>(o + j) = q;
        if constexpr (EPI == kBiasGelu) *reinterpret_cast<uint4*>(o2 + j) = q2;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < N; ++j) {
        const __nv_bfloat16 b = __float2bfloat16_rn(v[j]);
        o[j] = b;
        if constexpr (EPI == kBiasGelu) o2[j] = __float2bfloat16_rn(gelu_tanh(__bfloat162float(b)));
      }
    }
  }
}

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(256, 1)
    k_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const EpiArgs ep, int M, int N, int K) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n, num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&ta);
    ptx::tma_prefetch(&tb);
    for (int s = 0; s < C::kStages; ++s) ptx::mbar_init(&full[s], 1), ptx::mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) ptx::mbar_init(&tfull[a], 1), ptx::mbar_init(&tempty[a], 4);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, C::kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int mb = tile % num_m, nb = tile / num_m;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
          ptx::mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          if constexpr (!A_MN) {
            ptx::tma_load_2d(sa, &ta, &full[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              ptx::tma_load_2d(sa + c * (BK * 128), &ta, &full[stage], mb * BM + c * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            ptx::tma_load_2d(sb, &tb, &full[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              ptx::tma_load_2d(sb + c * (BK * 128), &tb, &full[stage], nb * BN + c * 64, kb * BK);
          }
          if (++stage == C::kStages) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        ptx::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + stage * C::kStageBytes);
          const uint32_t sb = sa + C::kABytes;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? ptx::smem_desc_sw128(sa + k * 2048, BK * 128, 1024)
                                     : ptx::smem_desc_sw128(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::smem_desc_sw128(sb + k * 2048, BK * 128, 1024)
                                     : ptx::smem_desc_sw128(sb + k * 32, 16, 1024);
            ptx::umma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == C::kStages) stage = 0, phase ^= 1;
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter owned by this warp
    int it = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const int mb = tile % num_m, nb = tile / num_m;
      ptx::mbar_wait(&tfull[acc], (it >> 1) & 1);
      ptx::tc_fence_after();
      const int row = mb * BM + q * 32 + lane;
      const uint32_t t0 = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(t0 + c * 32, r);
        ptx::tmem_ld_wait();
        const int col0 = nb * BN + c * 32;
        if (row < M && col0 < N) epilogue_chunk<EPI>(ep, row, col0, N, r);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void launch(int M, int N, int K, const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B,
            long long ldb, const EpiArgs& ep, cudaStream_t st) {
  using C = Cfg<BN>;
  const CUtensorMap ta = A_MN ? cuda::make_map_2d_bf16(A, M, K, lda, 64, BK)
                              : cuda::make_map_2d_bf16(A, K, M, lda, 64, BM);
  const CUtensorMap tb = B_MN ? cuda::make_map_2d_bf16(B, N, K, ldb, 64, BK)
                              : cuda::make_map_2d_bf16(B, K, N, ldb, 64, BN);
  auto kern = k_gemm<BN, A_MN, B_MN, EPI>;
  static bool attr = false;  // one-time per instantiation
  if (!attr) {
    CK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < cuda::kNumSMs ? tiles : cuda::kNumSMs;
  kern<<<grid, 256, C::kSmem, st>>>(ta, tb, ep, M, N, K);
  CK_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN>
void by_epi(Epi epi, int M, int N, int K, const __nv_bfloat16* A, long long lda,
            const __nv_bfloat16* B, long long ldb, const EpiArgs& ep, cudaStream_t st) {
  switch (epi) {
    case kStoreBF16: return launch<BN, A_MN, B_MN, kStoreBF16>(M, N, K, A, lda, B, ldb, ep, st);
    case kStoreF32: return launch<BN, A_MN, B_MN, kStoreF32>(M, N, K, A, lda, B, ldb, ep, st);
    case kAccF32: return launch<BN, A_MN, B_MN, kAccF32>(M, N, K, A, lda, B, ldb, ep, st);
    default: break;
  }
  if constexpr (!A_MN && !B_MN) {
    if (epi == kBiasGelu) return launch<BN, false, false, kBiasGelu>(M, N, K, A, lda, B, ldb, ep, st);
    if (epi == kBiasResid) return launch<BN, false, false, kBiasResid>(M, N, K, A, lda, B, ldb, ep, st);
  }
  if constexpr (!A_MN && B_MN) {
    if (epi == kGeluBwd) return launch<BN, false, true, kGeluBwd>(M, N, K, A, lda, B, ldb, ep, st);
  }
  throw chimera::capi::InternalError("gemm: unsupported epilogue/layout combination");
}

template <int BN>
void by_layout(Epi epi, bool a_mn, bool b_mn, int M, int N, int K, const __nv_bfloat16* A,
               long long lda, const __nv_bfloat16* B, long long ldb, const EpiArgs& ep,
               cudaStream_t st) {
  if (!a_mn && !b_mn) return by_epi<BN, false, false>(epi, M, N, K, A, lda, B, ldb, ep, st);
  if (!a_mn && b_mn) return by_epi<BN, false, true>(epi, M, N, K, A, lda, B, ldb, ep, st);
  if (a_mn && !b_mn) return by_epi<BN, true, false>(epi, M, N, K, A, lda, B, ldb, ep, st);
  return by_epi<BN, true, true>(epi, M, N, K, A, lda, B, ldb, ep, st);
}

}  // namespace

void gemm(Epi epi, bool a_mn, bool b_mn, int M, int N, int K, const __nv_bfloat16* A, long long lda,
          const __nv_bfloat16* B, long long ldb, const EpiArgs& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  if ((lda % 8) || (ldb % 8) || (reinterpret_cast<uintptr_t>(A) % 16) || (reinterpret_cast<uintptr_t>(B) % 16))
    throw chimera::capi::InternalError("gemm: operands must be 16-byte aligned with ld % 8 == 0");
  // 256-wide tiles when they still give at least one full wave of CTAs.
  const long long tiles256 = (long long)((M + BM - 1) / BM) * ((N + 255) / 256);
  if (N >= 256 && tiles256 >= cuda::kNumSMs)
    by_layout<256>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
  else
    by_layout<128>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
}

}  // namespace chimera::gemm

extern "C" {

// Test / integration entry: all pointers are device pointers; stream may be 0.
CK_API int ck_gemm_bf16(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A,
                        long long lda, const void* B, long long ldb, void* out, long long ldo,
                        const void* bias, const void* aux, long long ld_aux, void* out2,
                        long long ld_out2, void* stream) {
  return chimera::capi::guarded([&] {
    chimera::gemm::EpiArgs ep;
    ep.out = out;
    ep.ldo = ldo;
    ep.bias = static_cast<const __nv_bfloat16*>(bias);
    ep.aux = static_cast<const __nv_bfloat16*>(aux);
    ep.ld_aux = ld_aux;
    ep.out2 = static_cast<__nv_bfloat16*>(out2);
    ep.ld_out2 = ld_out2;
    chimera::gemm::gemm(static_cast<chimera::gemm::Epi>(epi), a_mn != 0, b_mn != 0, M, N, K,
                        static_cast<const __nv_bfloat16*>(A), lda, static_cast<const __nv_bfloat16*>(B),
                        ldb, ep, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
