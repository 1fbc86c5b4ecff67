// Persistent, warp-specialised tcgen05 GEMM for sm_100a with fused epilogues.
//
//   warp 0      TMA producer (one lane): K-blocks of A and B -> smem ring (mbarrier
//               full/empty), 128-byte swizzle, K-major or MN-major boxes
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16 128 x BN x 16 into one of
//               two TMEM accumulators; tcgen05.commit frees smem stages / hands the
//               finished accumulator to the epilogue
//   warp 2      TMEM allocator (2*BN fp32 columns)
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> swizzled smem
//               chunk -> TMA bulk tensor store (bf16) / reduce-add (fp32 accumulate);
//               a register epilogue with coalesced stores covers the other cases
// Double-buffered TMEM accumulators let tile i's epilogue overlap tile i+1's
// mainloop.  Grid = min(#tiles, 148): one resident CTA per SM.  The CTA-pair variant
// (k_gemm2, 256 x 256 tiles on tcgen05.mma.cta_group::2) carries most stage GEMMs;
// pick_tile chooses among the two by a calibrated wave model.
//
// This single kernel family serves every linear layer of the transformer stage:
// forward (A=X K-major, B=W K-major), activation gradient dX = dY W (B MN-major) and
// weight gradient dW += dY^T X (both operands MN-major), so no transpose is ever
// materialised in HBM.
#include <cuda.h>

#include <cstdlib>
#include <string>

#include "chimera_ck.h"
#include "common.cuh"
#include "gemm.cuh"
#include "ptx_sm100.cuh"
#include "tma_host.hpp"

namespace chimera::gemm {

// clock64() stamps per tile of CTA 0 (scripts/gemm_trace.cu builds with CK_GEMM_TRACE)
#ifdef CK_GEMM_TRACE
__device__ long long g_gemm_trace[16][8];
__device__ int g_gemm_trace_block = 0;
#define GEMM_TRACE(cond, t, ev)                                                                   \
  do {                                                                                            \
    if ((cond) && int(blockIdx.x) == g_gemm_trace_block && (t) < 16) g_gemm_trace[t][ev] = clock64(); \
  } while (0)
#else
#define GEMM_TRACE(cond, t, ev) \
  do {                          \
  } while (0)
#endif

namespace {

constexpr int BM = 128, BK = 64;

// Hardware tanh (one MUFU op, ~2^-11 relative error: below the bf16 output rounding).
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// Epilogue of one 32-row x 32-column accumulator chunk by one warp.  The tcgen05.ld
// 32x32b layout gives lane i row row0+i; the fp32 row is staged once through a padded
// per-warp smem tile and read back in "store layout" (lane <-> 8 consecutive bf16 or 4
// fp32 columns of one row), where bias / aux / accumulator operands -- prefetched into
// registers before the accumulator is even ready (EpiPre) -- are combined and written
// with fully coalesced 16-byte stores.
constexpr int kStgStride = 36;                         // floats per staged row (32 + 4 pad: conflict-free)
constexpr int kEpiWarpBytes = 32 * kStgStride * 4;     // 4608 B per epilogue warp

struct EpiPre {
  uint4 aux[4];   // bf16 aux rows (kBiasResid / kGeluBwd), store layout
  float4 acc[8];  // fp32 output rows (kAccF32), store layout
  uint4 bias;     // 8 bias values of this lane's columns
};

__device__ __forceinline__ float2 bf2f(uint32_t u) {
  return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
}
__device__ __forceinline__ uint32_t f2bf(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Output-tile order of the persistent loop: the tile index runs fastest over the
// dimension with fewer tiles, so one wave covers few blocks of the long operand, each
// shared by concurrently running tiles (read from HBM once) while the short operand
// stays L2-resident -- e.g. the LM-head weight gradient (50304 x 1024, K = tokens)
// would otherwise stream its 400 MB dlogits operand once per 256-column block.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int& mb, int& nb) {
  if (num_n <= num_m) {
    nb = tile % num_n;
    mb = (tile / num_n) % num_m;
  } else {
    mb = tile % num_m;
    nb = (tile / num_m) % num_n;
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue_prefetch(const EpiArgs& ep, int row0, int col0, int M, int N, int lane,
                                                  bool atomic, EpiPre& pre) {
  if constexpr (EPI == kAccF32) {
    if (atomic) return;
    const int col = col0 + (lane & 7) * 4;
    const float* out = static_cast<const float*>(ep.out);
    const bool vec = (N % 4) == 0 && (ep.ldo % 4) == 0 && col + 4 <= N;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int row = row0 + it * 4 + (lane >> 3);
      pre.acc[it] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row < M && vec) pre.acc[it] = *reinterpret_cast<const float4*>(out + (long long)row * ep.ldo + col);
    }
  } else if constexpr (EPI != kStoreF32) {
    const int col = col0 + (lane & 3) * 8;
    pre.bias = make_uint4(0, 0, 0, 0);
    if (ep.bias && EPI != kGeluBwd) {
      if ((N % 8) == 0 && col + 8 <= N) {
        pre.bias = *reinterpret_cast<const uint4*>(ep.bias + col);
      } else {
        __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&pre.bias);
        for (int t = 0; t < 8 && col + t < N; ++t) h[t] = ep.bias[col + t];
      }
    }
    if constexpr (EPI == kBiasResid || EPI == kGeluBwd) {
      const bool vec = (N % 8) == 0 && (ep.ld_aux % 8) == 0 && col + 8 <= N;
#pragma unroll
      for (int it = 0; it < 4; ++it) {
        const int row = row0 + it * 8 + (lane >> 2);
        uint4 q = make_uint4(0, 0, 0, 0);
        if (row < M && col < N) {
          const __nv_bfloat16* a = ep.aux + (long long)row * ep.ld_aux + col;
          if (vec) {
            q = *reinterpret_cast<const uint4*>(a);
          } else {
            __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&q);
            for (int t = 0; t < 8 && col + t < N; ++t) h[t] = a[t];
          }
        }
        pre.aux[it] = q;
      }
    }
  }
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const EpiArgs& ep, int row0, int col0, int M, int N,
                                               const uint32_t (&r)[32], uint8_t* stg_bytes, int lane, bool atomic,
                                               const EpiPre& pre) {
  float* stg = reinterpret_cast<float*>(stg_bytes);
#pragma unroll
  for (int j = 0; j < 32; j += 4)
    *reinterpret_cast<uint4*>(stg + lane * kStgStride + j) = make_uint4(r[j], r[j + 1], r[j + 2], r[j + 3]);
  __syncwarp();
  if constexpr (EPI == kAccF32 || EPI == kStoreF32) {
    float* out = static_cast<float*>(ep.out);
    const int sg = lane & 7, col = col0 + sg * 4;
    const bool vec = (N % 4) == 0 && (ep.ldo % 4) == 0 && col + 4 <= N;
#pragma unroll
    for (int it = 0; it < 8; ++it) {  // 32 rows x 8 segments of 4 floats
      const int rr = it * 4 + (lane >> 3), row = row0 + rr;
      if (row >= M || col >= N) continue;
      float4 x = *reinterpret_cast<const float4*>(stg + rr * kStgStride + sg * 4);
      float* o = out + (long long)row * ep.ldo + col;
      if (EPI == kAccF32 && atomic) {  // split-K partial sums
        if (vec) {
          atomicAdd(reinterpret_cast<float4*>(o), x);
        } else {
          const float xs[4] = {x.x, x.y, x.z, x.w};
          for (int t = 0; t < 4 && col + t < N; ++t) atomicAdd(o + t, xs[t]);
        }
      } else if (vec) {
        if constexpr (EPI == kAccF32) x.x += pre.acc[it].x, x.y += pre.acc[it].y, x.z += pre.acc[it].z, x.w += pre.acc[it].w;
        *reinterpret_cast<float4*>(o) = x;
      } else {
        const float xs[4] = {x.x, x.y, x.z, x.w};
        for (int t = 0; t < 4 && col + t < N; ++t) o[t] = (EPI == kAccF32 ? o[t] : 0.f) + xs[t];
      }
    }
  } else {
    const int sg = lane & 3, col = col0 + sg * 8;
    const bool vec_o = (N % 8) == 0 && (ep.ldo % 8) == 0 && col + 8 <= N;
    const bool vec_o2 = (N % 8) == 0 && (ep.ld_out2 % 8) == 0 && col + 8 <= N;
    float2 bias[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) bias[e] = bf2f((&pre.bias.x)[e]);
    float2 csum[4] = {};  // kGeluBwd + colsum: this lane's 8 columns over its rows
#pragma unroll
    for (int it = 0; it < 4; ++it) {  // 32 rows x 4 segments of 8 columns
      const int rr = it * 8 + (lane >> 2), row = row0 + rr;
      if (row >= M || col >= N) continue;
      const float4 x0 = *reinterpret_cast<const float4*>(stg + rr * kStgStride + sg * 8);
      const float4 x1 = *reinterpret_cast<const float4*>(stg + rr * kStgStride + sg * 8 + 4);
      float2 v[4] = {make_float2(x0.x, x0.y), make_float2(x0.z, x0.w), make_float2(x1.x, x1.y), make_float2(x1.z, x1.w)};
      if (EPI != kGeluBwd) {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = ptx::add2(v[e], bias[e]);
      }
      if constexpr (EPI == kBiasResid) {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = ptx::add2(v[e], bf2f((&pre.aux[it].x)[e]));
      }
      if constexpr (EPI == kGeluBwd) {  // v *= gelu_tanh'(u), u = aux
        const float k0 = 0.7978845608028654f, k1 = 0.044715f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 u = bf2f((&pre.aux[it].x)[e]);
          const float2 u2 = ptx::mul2(u, u);
          const float2 z = ptx::mul2(u, ptx::fma2(u2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0)));
          const float2 t = make_float2(tanh_fast(z.x), tanh_fast(z.y));
          const float2 a = ptx::fma2(t, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
          const float2 om = ptx::fma2(make_float2(-t.x, -t.y), t, make_float2(1.f, 1.f));
          const float2 c = ptx::fma2(u2, make_float2(3.f * k0 * k1, 3.f * k0 * k1), make_float2(k0, k0));
          const float2 hb = ptx::mul2(ptx::mul2(u, make_float2(0.5f, 0.5f)), om);
          v[e] = ptx::mul2(v[e], ptx::fma2(hb, c, a));
        }
      }
      uint4 q;
      q.x = f2bf(v[0].x, v[0].y), q.y = f2bf(v[1].x, v[1].y), q.z = f2bf(v[2].x, v[2].y), q.w = f2bf(v[3].x, v[3].y);
      if constexpr (EPI == kGeluBwd) {
        if (ep.colsum) {
#pragma unroll
          for (int e = 0; e < 4; ++e) csum[e] = ptx::add2(csum[e], bf2f((&q.x)[e]));
        }
      }
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + col;
      if (vec_o) {
        *reinterpret_cast<uint4*>(dst) = q;
      } else {
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q);
        for (int t = 0; t < 8 && col + t < N; ++t) dst[t] = h[t];
      }
      if constexpr (EPI == kBiasGelu) {  // G = gelu_tanh(U) of the bf16-rounded U
        const float k0 = 0.7978845608028654f, k1 = 0.044715f;
        uint4 g;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 u = bf2f((&q.x)[e]);
          const float2 u2 = ptx::mul2(u, u);
          const float2 z = ptx::mul2(u, ptx::fma2(u2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0)));
          const float2 t = make_float2(tanh_fast(z.x), tanh_fast(z.y));
          const float2 hu = ptx::mul2(u, make_float2(0.5f, 0.5f));
          const float2 y = ptx::fma2(hu, t, hu);
          (&g.x)[e] = f2bf(y.x, y.y);
        }
        __nv_bfloat16* dst2 = ep.out2 + (long long)row * ep.ld_out2 + col;
        if (vec_o2) {
          *reinterpret_cast<uint4*>(dst2) = g;
        } else {
          const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&g);
          for (int t = 0; t < 8 && col + t < N; ++t) dst2[t] = h[t];
        }
      }
    }
    if constexpr (EPI == kGeluBwd) {
      if (ep.colsum) {  // reduce over the 8 lanes sharing these columns, one atomic per column
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            csum[e].x += __shfl_xor_sync(0xffffffffu, csum[e].x, off);
            csum[e].y += __shfl_xor_sync(0xffffffffu, csum[e].y, off);
          }
        if (lane < 4 && col < N) {
          if ((N % 8) == 0 && col + 8 <= N) {
            float4* d = reinterpret_cast<float4*>(ep.colsum + col);
            atomicAdd(d, make_float4(csum[0].x, csum[0].y, csum[1].x, csum[1].y));
            atomicAdd(d + 1, make_float4(csum[2].x, csum[2].y, csum[3].x, csum[3].y));
          } else {
            for (int t = 0; t < 8 && col + t < N; ++t) atomicAdd(ep.colsum + col + t, (&csum[t >> 1].x)[t & 1]);
          }
        }
      }
    }
  }
  __syncwarp();
}

// TMA-store epilogue (every bf16 output epilogue, and kAccF32) of one 32 x 32 accumulator chunk in the
// tcgen05.ld layout (lane = row, 32 consecutive fp32 columns): the warp writes it to its
// swizzled smem staging and one lane issues a bulk tensor store (bf16, 64-byte swizzle,
// two alternating 2 KB buffers) or a bulk tensor reduce-add (fp32 += D at L2: the weight-
// gradient accumulate, split-K included, with no read-back of the output) -- no
// shared-memory round trip to a store layout, no per-thread global stores, and the
// stores drain asynchronously while the next chunk (or tile) proceeds.
// The residual operand of a kBiasResid chunk in the same layout: this lane's row, 32
// columns (four 16-byte loads), fetched one chunk ahead.
template <int EPI>
__device__ __forceinline__ void aux_row_prefetch(const EpiArgs& ep, int row, int col0, int M, int N, uint4 (&a)[4]) {
  if constexpr (EPI == kBiasResid || EPI == kGeluBwd) {
    const bool ok = row < M && col0 < N;  // N % 32 == 0 on this path: whole chunks
    const __nv_bfloat16* p = ep.aux + (long long)row * ep.ld_aux + col0;
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = ok ? *reinterpret_cast<const uint4*>(p + 8 * k) : make_uint4(0, 0, 0, 0);
  }
}

// The chunk's 32 bias values as bf16 pairs, pair i in lane i (broadcast by shuffles in
// the epilogue): one 4-byte load per lane, issued a chunk ahead like the residual rows.
__device__ __forceinline__ uint32_t bias_prefetch(const EpiArgs& ep, int col0, int N, int lane) {
  if (!ep.bias || lane >= 16 || col0 >= N) return 0u;
  return *reinterpret_cast<const uint32_t*>(ep.bias + col0 + 2 * lane);
}

template <int EPI>
__device__ __forceinline__ void epilogue_chunk_tma(const EpiArgs& ep, const CUtensorMap* to, const CUtensorMap* to2,
                                                   int row0, int col0, const uint32_t (&r)[32], uint8_t* stg,
                                                   int lane, int& nbuf, const uint4 (&aux)[4], uint32_t bias2) {
  if constexpr (EPI == kAccF32) {
    if (lane == 0) ptx::bulk_wait_read0();  // the previous reduce has read the staging
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(stg + lane * 128 + ((j ^ (lane & 7)) << 4)) =
          make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
    ptx::fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_reduce_add_2d(to, stg, col0, row0);
      ptx::bulk_commit();
    }
  } else {
    uint32_t q[16];
    if (ep.bias) {  // the chunk's 32 bias values: pair i from lane i
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float2 bb = bf2f(__shfl_sync(0xffffffffu, bias2, i));
        if constexpr (EPI == kBiasResid) bb = ptx::add2(bb, bf2f((&aux[i >> 2].x)[i & 3]));
        q[i] = f2bf(__uint_as_float(r[2 * i]) + bb.x, __uint_as_float(r[2 * i + 1]) + bb.y);
      }
    } else if constexpr (EPI == kBiasResid) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 a = bf2f((&aux[i >> 2].x)[i & 3]);
        q[i] = f2bf(__uint_as_float(r[2 * i]) + a.x, __uint_as_float(r[2 * i + 1]) + a.y);
      }
    } else if constexpr (EPI == kGeluBwd) {  // D * gelu_tanh'(U), U = aux
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 u = bf2f((&aux[i >> 2].x)[i & 3]);
        const float2 u2 = ptx::mul2(u, u);
        const float2 z = ptx::mul2(u, ptx::fma2(u2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0)));
        const float2 t = make_float2(tanh_fast(z.x), tanh_fast(z.y));
        const float2 a = ptx::fma2(t, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
        const float2 om = ptx::fma2(make_float2(-t.x, -t.y), t, make_float2(1.f, 1.f));
        const float2 c = ptx::fma2(u2, make_float2(3.f * k0 * k1, 3.f * k0 * k1), make_float2(k0, k0));
        const float2 hb = ptx::mul2(ptx::mul2(u, make_float2(0.5f, 0.5f)), om);
        const float2 v = ptx::mul2(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])),
                                   ptx::fma2(hb, c, a));
        q[i] = f2bf(v.x, v.y);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) q[i] = f2bf(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
    }
    uint8_t* buf = stg + (nbuf & 1) * 2048;
    // the stores issued from these buffers two chunks ago have read them (one bulk group
    // per chunk: U alone, or U + G)
    if (lane == 0) ptx::bulk_wait_read1();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<uint4*>(buf + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
          make_uint4(q[4 * j], q[4 * j + 1], q[4 * j + 2], q[4 * j + 3]);
    if constexpr (EPI == kBiasGelu) {  // G = gelu_tanh(U) of the bf16-rounded U
      const float k0 = 0.7978845608028654f, k1 = 0.044715f;
      uint32_t gq[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 u = bf2f(q[i]);
        const float2 u2 = ptx::mul2(u, u);
        const float2 z = ptx::mul2(u, ptx::fma2(u2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0)));
        const float2 t = make_float2(tanh_fast(z.x), tanh_fast(z.y));
        const float2 hu = ptx::mul2(u, make_float2(0.5f, 0.5f));
        const float2 y = ptx::fma2(hu, t, hu);
        gq[i] = f2bf(y.x, y.y);
      }
      uint8_t* buf2 = buf + 4096;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<uint4*>(buf2 + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
            make_uint4(gq[4 * j], gq[4 * j + 1], gq[4 * j + 2], gq[4 * j + 3]);
    }
    ptx::fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      ptx::tma_store_2d(to, buf, col0, row0);
      if constexpr (EPI == kBiasGelu) ptx::tma_store_2d(to2, buf + 4096, col0, row0);
      ptx::bulk_commit();
    }
    if constexpr (EPI == kGeluBwd) {
      if (ep.colsum) {  // the fused bias gradient: lane sums its column of the staged bf16 chunk
        float cs = 0.f;
#pragma unroll 8
        for (int rr = 0; rr < 32; ++rr)
          cs += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
              buf + rr * 64 + ((((lane >> 3) ^ ((rr >> 1) & 3))) << 4) + (lane & 7) * 2));
        atomicAdd(ep.colsum + col0 + lane, cs);  // rows past M: zero-filled A rows and aux -> 0
      }
    }
    ++nbuf;
  }
}

template <int BN>
struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kStgBytes = 8192;  // per epilogue warp, 1 KB aligned (TMA-store layouts)
  static constexpr int kSmem = kStages * kStageBytes + 4 * kStgBytes + 256 + 1024;
};

template <int BN, bool A_MN, bool B_MN, int EPI, bool TO>
__global__ void __launch_bounds__(256, 1)
    k_gemm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const __grid_constant__ CUtensorMap to, const __grid_constant__ CUtensorMap to2, const EpiArgs ep, int M,
           int N, int K, int ksplit) {
  static_assert(!TO || EPI != kStoreF32, "TMA-store epilogue: bf16 outputs / fp32 accumulate");
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB aligned (128-byte swizzle atoms); pointer arithmetic on the __shared__ array keeps
  // the state space visible, so the epilogue staging compiles to STS/LDS, not generic ST/LD
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stg_base = smem + C::kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_base + 4 * C::kStgBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int num_kb = (K + BK - 1) / BK, kb_per = (num_kb + ksplit - 1) / ksplit;
  const int tiles = num_m * num_n * ksplit;

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
  cuda::pdl_wait();     // operands / outputs of the previous kernel in the stream
  cuda::pdl_trigger();  // persistent grid: successors may be scheduled on free SMs

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        const int ks = tile / (num_m * num_n);
        const int kb1 = min(num_kb, (ks + 1) * kb_per);
        for (int kb = ks * kb_per; kb < kb1; ++kb) {
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
        const int ks = tile / (num_m * num_n);
        const int kb0 = ks * kb_per, kb1 = min(num_kb, (ks + 1) * kb_per);
        for (int kb = kb0; kb < kb1; ++kb) {
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
            ptx::umma_f16(d_tmem, ad, bd, idesc, (kb > kb0 || k) ? 1u : 0u);
          }
          ptx::umma_commit(&empty[stage]);
          if (++stage == C::kStages) stage = 0, phase ^= 1;
        }
        ptx::umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp - 4;  // TMEM lane quarter owned by this warp
    uint8_t* stg = stg_base + q * C::kStgBytes;
    int it = 0, nbuf = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int row0 = mb * BM + q * 32;
      EpiPre pre;
      uint4 auxn[4], auxn2[4];  // residual / U rows of the next two chunks (TMA epilogue)
      if constexpr (!TO) {
        epilogue_prefetch<EPI>(ep, row0, nb * BN, M, N, lane, (ksplit > 1 || ep.atomic_acc), pre);
      } else {
        aux_row_prefetch<EPI>(ep, row0 + lane, nb * BN, M, N, auxn);
        if (BN / 32 > 1) aux_row_prefetch<EPI>(ep, row0 + lane, nb * BN + 32, M, N, auxn2);
      }
      uint32_t biasn = TO ? bias_prefetch(ep, nb * BN, N, lane) : 0u;
      ptx::mbar_wait(&tfull[acc], (it >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t t0 = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(t0 + c * 32, r);
        const int col0 = nb * BN + c * 32;
        if constexpr (TO) {
          uint4 auxc[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) auxc[k] = auxn[k], auxn[k] = auxn2[k];
          if (c + 2 < BN / 32) aux_row_prefetch<EPI>(ep, row0 + lane, col0 + 64, M, N, auxn2);
          const uint32_t biasc = biasn;
          if (c + 1 < BN / 32) biasn = bias_prefetch(ep, col0 + 32, N, lane);
          ptx::tmem_ld_wait();
          if (row0 < M && col0 < N)
            epilogue_chunk_tma<EPI>(ep, &to, &to2, row0, col0, r, stg, lane, nbuf, auxc, biasc);
        } else {
          EpiPre cur = pre;
          if (c + 1 < BN / 32) epilogue_prefetch<EPI>(ep, row0, col0 + 32, M, N, lane, (ksplit > 1 || ep.atomic_acc), pre);
          ptx::tmem_ld_wait();
          if (row0 < M && col0 < N) epilogue_chunk<EPI>(ep, row0, col0, M, N, r, stg, lane, (ksplit > 1 || ep.atomic_acc), cur);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
    }
    if constexpr (TO)
      if (lane == 0) ptx::bulk_wait0();
  }
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem_base, C::kTmemCols);
  }
}

// Split-K for the fp32-accumulate (weight-gradient) epilogue when the output tiles alone
// cannot fill the machine: the smallest slice count (each >= 8 K-blocks deep) whose
// last wave is (nearly) as full as the best achievable; slices combine with fp32 vector
// atomics.
inline int split_k(int epi, int tiles, int slots, int K, int chosen = 0) {
  static const int force = [] {  // CK_GEMM_KSPLIT=n: fixed slice count (benchmarks)
    const char* e = std::getenv("CK_GEMM_KSPLIT");
    return e ? atoi(e) : 0;
  }();
  if (chosen > 0) return chosen;
  if (epi == kAccF32 && force > 0) return force;
  if (epi != kAccF32) return 1;
  const int kb = (K + BK - 1) / BK;
  if (tiles >= slots) {
    // more than one wave: two slices when they cut the waves x depth product by >= 20 %
    // (e.g. 75 or 100 CTA-pair tiles on 74 pairs: the weight gradients of GPT-2 1.3B's
    // QKV / FC layers) -- more slices only add fp32 read-modify-write traffic to the
    // HBM-resident gradient (graph-timed sweep, profiles/r02r_wgrad_sweep.jsonl)
    const long long w1 = (long long)((tiles + slots - 1) / slots) * kb;
    const long long w2 = (long long)((2LL * tiles + slots - 1) / slots) * ((kb + 1) / 2);
    return (kb >= 16 && w2 * 5 <= w1 * 4) ? 2 : 1;
  }
  // (more than 4 slices: the extra fp32 atomic traffic costs more than the wave it fills)
  const int kmax = kb / 8 < 1 ? 1 : (kb / 8 > 4 ? 4 : kb / 8);
  auto eff = [&](int ks) {
    const long long u = (long long)tiles * ks, waves = (u + slots - 1) / slots;
    return double(u) / double(waves * slots);
  };
  double best = 0.0;
  for (int ks = 1; ks <= kmax; ++ks) best = eff(ks) > best ? eff(ks) : best;
  for (int ks = 1; ks <= kmax; ++ks)
    if (eff(ks) >= best - 0.03) return ks;
  return 1;
}


// ------------------------------------------------ split-K for bf16 epilogues --
// Problems whose output tiles cannot fill 148 SMs (the 632 / 1264-row stage GEMMs of
// GPT-2 1.3B with N = h, deep K) run as K-slices: every slice reduce-adds its fp32
// partial tile into a zero-filled workspace (the kAccF32 kernels, TMA bulk reduce-add
// at L2), then this pass applies the epilogue to the reduced rows with the arithmetic
// of epilogue_chunk_tma (bias + residual summed first, gelu_tanh / gelu_tanh' on the
// same formulas, bf16 rounding, the fused bias-gradient column sums of the bf16
// values), writes the outputs and re-zeroes the workspace for the stream's next call.
// Thread = 8 consecutive columns x kFinRows rows (16-byte loads and stores).
constexpr int kFinRows = 8;

template <int EPI>
__global__ void __launch_bounds__(128) k_splitk_finalize(float* __restrict__ ws, EpiArgs ep, int M, int N) {
  cuda::pdl_wait();  // launched with programmatic serialisation: the slices must have landed
  const int col = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (col >= N) return;
  const int row0 = blockIdx.y * kFinRows;
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float2 bias[4] = {};
  if (ep.bias && EPI != kGeluBwd) {
    const uint4 b = *reinterpret_cast<const uint4*>(ep.bias + col);
#pragma unroll
    for (int e = 0; e < 4; ++e) bias[e] = bf2f((&b.x)[e]);
  }
  float2 csum[4] = {};
  for (int rr = 0; rr < kFinRows; ++rr) {
    const int row = row0 + rr;
    if (row >= M) break;
    float4* src = reinterpret_cast<float4*>(ws + (long long)row * N + col);
    const float4 x0 = src[0], x1 = src[1];
    src[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    src[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    float2 v[4] = {make_float2(x0.x, x0.y), make_float2(x0.z, x0.w), make_float2(x1.x, x1.y), make_float2(x1.z, x1.w)};
    uint4 q;
    if constexpr (EPI == kGeluBwd) {
      const uint4 a = *reinterpret_cast<const uint4*>(ep.aux + (long long)row * ep.ld_aux + col);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 u = bf2f((&a.x)[e]);
        const float2 u2 = ptx::mul2(u, u);
        const float2 z = ptx::mul2(u, ptx::fma2(u2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0)));
        const float2 t = make_float2(tanh_fast(z.x), tanh_fast(z.y));
        const float2 g = ptx::fma2(t, make_float2(0.5f, 0.5f), make_float2(0.5f, 0.5f));
        const float2 om = ptx::fma2(make_float2(-t.x, -t.y), t, make_float2(1.f, 1.f));
        const float2 c = ptx::fma2(u2, make_float2(3.f * k0 * k1, 3.f * k0 * k1), make_float2(k0, k0));
        const float2 hb = ptx::mul2(ptx::mul2(u, make_float2(0.5f, 0.5f)), om);
        const float2 y = ptx::mul2(v[e], ptx::fma2(hb, c, g));
        (&q.x)[e] = f2bf(y.x, y.y);
        if (ep.colsum) csum[e] = ptx::add2(csum[e], bf2f((&q.x)[e]));
      }
    } else {
      uint4 a = make_uint4(0, 0, 0, 0);
      if constexpr (EPI == kBiasResid) a = *reinterpret_cast<const uint4*>(ep.aux + (long long)row * ep.ld_aux + col);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float2 bb = bias[e];
        if constexpr (EPI == kBiasResid) bb = ep.bias ? ptx::add2(bb, bf2f((&a.x)[e])) : bf2f((&a.x)[e]);
        (&q.x)[e] = (ep.bias || EPI == kBiasResid) ? f2bf(v[e].x + bb.x, v[e].y + bb.y) : f2bf(v[e].x, v[e].y);
      }
    }
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(ep.out) + (long long)row * ep.ldo + col) = q;
    if constexpr (EPI == kBiasGelu) {  // G = gelu_tanh(U) of the bf16-rounded U
      uint4 gq;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 u = bf2f((&q.x)[e]);
        const float2 u2 = ptx::mul2(u, u);
        const float2 z = ptx::mul2(u, ptx::fma2(u2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0)));
        const float2 t = make_float2(tanh_fast(z.x), tanh_fast(z.y));
        const float2 hu = ptx::mul2(u, make_float2(0.5f, 0.5f));
        const float2 y = ptx::fma2(hu, t, hu);
        (&gq.x)[e] = f2bf(y.x, y.y);
      }
      *reinterpret_cast<uint4*>(ep.out2 + (long long)row * ep.ld_out2 + col) = gq;
    }
  }
  if constexpr (EPI == kGeluBwd) {
    if (ep.colsum) {
      float4* d = reinterpret_cast<float4*>(ep.colsum + col);
      atomicAdd(d, make_float4(csum[0].x, csum[0].y, csum[1].x, csum[1].y));
      atomicAdd(d + 1, make_float4(csum[2].x, csum[2].y, csum[3].x, csum[3].y));
    }
  }
}

// ------------------------------------------------------------------ stream-K --
// The CTA-pair kernel's work list.  Classic: output tiles pair, pair + npairs, ... (each
// split into ksplit K-slices).  Stream-K (`sk` != 0): the tiles x K-blocks iteration
// space is cut into npairs equal contiguous ranges, so no pair idles in a partial last
// wave (50 tiles on 74 pairs: the N = 1280 stage GEMMs of GPT-2 1.3B at 2528 rows; 150
// or 200 tiles: 2.03 / 2.7 waves).  A pair visits its range in DECREASING tile order:
// its first item -- the head of the tile its range ends in -- is a PARTIAL (fp32 tile to
// the workspace slot of this pair, then a per-CTA flag), its last item -- the tail of
// the tile its range starts in -- OWNS that tile: it waits for the partials of the
// lower-numbered pairs sharing the tile (already written: they were those pairs' first
// items, and lower block indices are scheduled first), adds them and runs the fused
// epilogue.  fp32 accumulate (weight gradients) needs no fix-up: every segment
// reduce-adds its own part.
struct SkItem {
  int tile = 0, ks = 0, kb0 = 0, kb1 = 0;
  bool partial = false;  // write the fp32 partial, no epilogue
  bool fixup = false;    // add the partials of lower pairs before the epilogue
};
struct WorkList {
  int pair, npairs, tiles, num_kb, kb_per, ksplit;
  bool sk, acc;  // stream-K; fp32 accumulate (segments reduce-add, no fix-up)
  long long b = 0, e = 0, cur = 0;
  int next_tile = 0;
  __device__ void init(int pair_, int npairs_, int base_tiles, int num_kb_, int ksplit_, bool sk_, bool acc_) {
    pair = pair_, npairs = npairs_, num_kb = num_kb_, ksplit = ksplit_, sk = sk_, acc = acc_;
    tiles = base_tiles * (sk ? 1 : ksplit);
    kb_per = (num_kb + ksplit - 1) / ksplit;
    if (sk) {
      const long long T = (long long)base_tiles * num_kb;
      b = T * pair / npairs, e = T * (pair + 1) / npairs, cur = e;
    } else {
      next_tile = pair;
    }
  }
  __device__ bool next(SkItem& it) {
    if (!sk) {
      if (next_tile >= tiles) return false;
      it.tile = next_tile % (tiles / ksplit);
      it.ks = next_tile / (tiles / ksplit);
      it.kb0 = it.ks * kb_per;
      it.kb1 = min(num_kb, it.kb0 + kb_per);
      it.partial = it.fixup = false;
      next_tile += npairs;
      return true;
    }
    if (cur <= b) return false;
    const long long last = cur - 1;  // the highest remaining iteration
    const int t = int(last / num_kb);
    const long long t0 = (long long)t * num_kb;
    const long long lo = t0 > b ? t0 : b;
    it.tile = t, it.ks = 0, it.kb0 = int(lo - t0), it.kb1 = int(cur - t0);
    it.partial = !acc && it.kb1 < num_kb;                  // lacks the tile's last K-block
    it.fixup = !acc && !it.partial && it.kb0 > 0;          // has it, but not the first
    cur = lo;
    return true;
  }
  // the pairs (below `pair`) holding the other segments of the tile this pair owns
  __device__ int first_producer(int t) const {  // lowest pair index whose range meets tile t
    const long long T = (long long)tiles * num_kb, t0 = (long long)t * num_kb;
    int q = pair;
    while (q > 0 && T * q / npairs > t0) --q;  // range of q starts after t0 -> q-1 also in t
    return q;
  }
};
constexpr int kSkFlagInts = 2 * 160;  // per (pair, CTA) completion counters at the workspace tail

// ---------------------------------------------------------- 2-SM variant ----
// A CTA pair (cluster of 2 on one TPC) computes a 256 x PBN tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its 128 rows of A and PBN/2 of
// the PBN rows of B per K-block, so per-SM operand traffic per MMA drops versus a
// single-CTA tile.  The leader (even) CTA issues the MMAs and owns the smem-full and
// TMEM-empty barriers; commits are multicast to both CTAs.  PBN = 256 is the one used:
// a 256 x 128 tile (two per pair on the single-wave stage shapes, the first epilogue
// under the second mainloop) measured 0.6-0.7x of it on every stage shape -- per-SM
// operand traffic per MMA grows by half and the mainloop becomes operand-bound.
constexpr int kPairEpiWarps = 8;  // two per TMEM lane quarter, each owning half of the columns
// AUX: the bias+residual TMA epilogue stages each warp's 32 x 128 residual block in shared
// memory with one TMA load issued under the mainloop (4-stage ring to make room).
template <int PBN, bool AUX = false>
struct PairCfg {
  static constexpr int kABytes = 128 * BK * 2;               // this CTA's 128 rows of A
  static constexpr int kBBytes = (PBN / 2) * BK * 2;         // this CTA's PBN/2 rows of B
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = AUX ? 4 : PBN >= 192 ? 5 : 7;
  static constexpr int kTmemCols = 2 * PBN <= 256 ? 256 : 512;  // two accumulators, power of 2
  // per-warp epilogue staging, 1 KB aligned for the swizzled TMA-store layouts: 2 x (U, G)
  // 2 KB bf16 chunk buffers; when AUX, 2 x 2 KB output buffers + the 8 KB residual block
  static constexpr int kAuxOff = 4096;
  static constexpr int kStgBytes = AUX ? 4096 + 8192 : 8192;
  static_assert(kStgBytes >= kEpiWarpBytes, "staging");
  static constexpr int kSmem = kStages * kStageBytes + kPairEpiWarps * kStgBytes + 256 + 1024;
  static_assert(kSmem <= 227 * 1024, "shared memory");
  static constexpr int kChunks = PBN / 64;                   // 32-column chunks per epilogue warp
};

template <int PBN, bool A_MN, bool B_MN, int EPI, bool TO>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 32 * kPairEpiWarps, 1)
    k_gemm2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
            const __grid_constant__ CUtensorMap to, const __grid_constant__ CUtensorMap to2, const EpiArgs ep,
            int M, int N, int K, int ksplit, int sk) {
  static_assert(!TO || EPI != kStoreF32, "TMA-store epilogue: bf16 outputs / fp32 accumulate");
  constexpr bool AUX = TO && EPI == kBiasResid;  // residual block via TMA (tensor map `to2`)
  using C = PairCfg<PBN, AUX>;
  extern __shared__ uint8_t smem_raw[];
  GEMM_TRACE(threadIdx.x == 32, 0, 6);
  // 1 KB aligned (128-byte swizzle atoms); pointer arithmetic on the __shared__ array keeps
  // the state space visible, so the epilogue staging compiles to STS/LDS, not generic ST/LD
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stg_base = smem + C::kStages * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stg_base + kPairEpiWarps * C::kStgBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* auxbar = tempty + 2;  // [kPairEpiWarps] residual block landed (AUX)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(auxbar + kPairEpiWarps);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cta = ptx::cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_m = (M + 255) / 256, num_n = (N + PBN - 1) / PBN;
  const int num_kb = (K + BK - 1) / BK;
  WorkList wl0;  // this pair's work items (classic tiles or a stream-K range)
  wl0.init(pair, npairs, num_m * num_n, num_kb, ksplit, sk != 0, EPI == kAccF32);

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&ta);
    ptx::tma_prefetch(&tb);
    if constexpr (TO) ptx::tma_prefetch(&to);
    if constexpr (TO && EPI == kBiasGelu) ptx::tma_prefetch(&to2);
    for (int s = 0; s < C::kStages; ++s) ptx::mbar_init(&full[s], 1), ptx::mbar_init(&empty[s], 1);
    for (int a = 0; a < 2; ++a) ptx::mbar_init(&tfull[a], 1), ptx::mbar_init(&tempty[a], 2 * kPairEpiWarps);
    for (int w = 0; w < kPairEpiWarps; ++w) ptx::mbar_init(&auxbar[w], 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc2(tmem_slot, C::kTmemCols);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  cuda::pdl_wait();
  cuda::pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      WorkList wl = wl0;
      for (SkItem itm; wl.next(itm);) {
        int mb, nb;
        tile_coords(itm.tile, num_m, num_n, mb, nb);
        const int m0 = mb * 256 + int(cta) * 128, n0 = nb * PBN + int(cta) * (PBN / 2);
        for (int kb = itm.kb0; kb < itm.kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::kStageBytes;
          uint8_t* sb = sa + C::kABytes;
#ifdef CK_GEMM_NOFEED  // scripts/gemm_trace.cu: the MMA rate with no operand traffic (timing only)
          if (cta == 0) ptx::mbar_arrive(&full[stage]);
          if (++stage == C::kStages) stage = 0, phase ^= 1;
          continue;
#endif
          if (cta == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * C::kStageBytes);
          if constexpr (!A_MN) {
            ptx::tma_load_2d_pair(sa, &ta, &full[stage], kb * BK, m0);
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) ptx::tma_load_2d_pair(sa + c * (BK * 128), &ta, &full[stage], m0 + c * 64, kb * BK);
          }
          if constexpr (!B_MN) {
            ptx::tma_load_2d_pair(sb, &tb, &full[stage], kb * BK, n0);
          } else {
#pragma unroll
            for (int c = 0; c < PBN / 128; ++c)
              ptx::tma_load_2d_pair(sb + c * (BK * 128), &tb, &full[stage], n0 + c * 64, kb * BK);
          }
          if (++stage == C::kStages) stage = 0, phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (cta == 0 && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16(256, PBN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      WorkList wl = wl0;
      for (SkItem itm; wl.next(itm); ++it) {
        const int acc = it & 1;
        ptx::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        GEMM_TRACE(true, it, 0);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * PBN;
        const int kb0 = itm.kb0, kb1 = itm.kb1;
        for (int kb = kb0; kb < kb1; ++kb) {
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
            ptx::umma_f16_pair(d_tmem, ad, bd, idesc, (kb > kb0 || k) ? 1u : 0u);
          }
          ptx::umma_commit_pair(&empty[stage]);
          if (++stage == C::kStages) stage = 0, phase ^= 1;
        }
        GEMM_TRACE(true, it, 1);
        ptx::umma_commit_pair(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3, half = (warp - 4) >> 2;  // lane quarter, column half
    constexpr int NC = C::kChunks;
    uint8_t* stg = stg_base + (warp - 4) * C::kStgBytes;
    int it = 0, nbuf = 0, aux_it = 0;
    // stream-K fix-up state: this pair's fp32 partial slot (this CTA's 128 rows) and the
    // per-(pair, CTA) completion counters at the workspace tail
    float* const slot_base = ep.ws;
    int* const flags = sk ? reinterpret_cast<int*>(ep.ws + ep.ws_elems) - kSkFlagInts : nullptr;
    auto slot_of = [&](int pq) { return slot_base + (size_t(pq) * 2 + cta) * (128 * PBN); };
    WorkList wl = wl0;
    for (SkItem itm; wl.next(itm); ++it) {
      const int acc = it & 1;
      int mb, nb;
      tile_coords(itm.tile, num_m, num_n, mb, nb);
      if (itm.partial) {  // stream-K head / middle segment: fp32 partial -> workspace slot
        ptx::mbar_wait(&tfull[acc], (it >> 1) & 1);
        GEMM_TRACE(warp == 4 && lane == 0, it, 2);  // partial: accumulator ready
        ptx::tc_fence_after();
        const uint32_t tp = tmem_base + (uint32_t(q * 32) << 16) + acc * PBN;
        // warp-interleaved layout: for each (chunk, 16-byte piece k) the 32 lanes' pieces
        // are contiguous, so every store instruction writes 512 B in full sectors (a
        // row-major slot made each instruction 32 partial-sector writes: ~10 us per tile)
        float* sw = slot_of(pair) + size_t((q * 2 + half) * NC) * 32 * 32;
#pragma unroll 1
        for (int c = half * NC; c < half * NC + NC; ++c) {
          uint32_t r[32];
          ptx::tmem_ld32(tp + c * 32, r);
          ptx::tmem_ld_wait();
          float* sc = sw + size_t(c - half * NC) * 32 * 32;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            *reinterpret_cast<uint4*>(sc + (k * 32 + lane) * 4) = make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_leader_relaxed(&tempty[acc]);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(flags + pair * 2 + int(cta), 1);
        GEMM_TRACE(warp == 4 && lane == 0, it, 3);  // partial stored + published
        continue;
      }
      int q_lo = pair;  // fix-up: partials of pairs [q_lo, pair) of this tile
      if (itm.fixup) q_lo = wl.first_producer(itm.tile);
      EpiPre pre;  // this tile's first-chunk operands are fetched while the MMAs run
      uint4 auxn[4], auxn2[4];  // residual / U rows of the next two chunks (TMA epilogue), in
                                // flight under the mainloop: their HBM latency is what the
                                // single-wave shapes' exposed epilogue otherwise waits on
      if constexpr (!TO) {
        epilogue_prefetch<EPI>(ep, mb * 256 + int(cta) * 128 + q * 32, nb * PBN + half * (PBN / 2), M, N, lane,
                               (ksplit > 1 || sk || ep.atomic_acc), pre);
      } else if constexpr (AUX) {  // this warp's residual block, one TMA box per chunk
        ptx::fence_proxy_async();  // the previous tile's reads of the block precede the refill
        __syncwarp();
        if (lane == 0) {
          const int rw = mb * 256 + int(cta) * 128 + q * 32, c0 = nb * PBN + half * (PBN / 2);
          ptx::mbar_arrive_expect_tx(&auxbar[warp - 4], NC * 2048);
          for (int c = 0; c < NC; ++c)
            ptx::tma_load_2d(stg + C::kAuxOff + c * 2048, &to2, &auxbar[warp - 4], c0 + 32 * c, rw);
        }
        ++aux_it;
      } else {
        const int rr = mb * 256 + int(cta) * 128 + q * 32 + lane, c0 = nb * PBN + half * (PBN / 2);
        aux_row_prefetch<EPI>(ep, rr, c0, M, N, auxn);
        if (NC > 1) aux_row_prefetch<EPI>(ep, rr, c0 + 32, M, N, auxn2);
      }
      uint32_t biasn = TO ? bias_prefetch(ep, nb * PBN + half * (PBN / 2), N, lane) : 0u;
      ptx::mbar_wait(&tfull[acc], (it >> 1) & 1);
      GEMM_TRACE(warp == 4 && lane == 0, it, 2);
      GEMM_TRACE(warp == 11 && lane == 0, it, 4);
      ptx::tc_fence_after();
      if (itm.fixup) {  // the lower pairs' partials of this tile have landed (8 warps each)
        if (lane == 0)
          for (int pq = q_lo; pq < pair; ++pq)
            while (*reinterpret_cast<volatile int*>(flags + pq * 2 + int(cta)) < kPairEpiWarps) __nanosleep(32);
        __syncwarp();
        __threadfence();
        GEMM_TRACE(warp == 4 && lane == 0, it, 7);
      }
      const int row0 = mb * 256 + int(cta) * 128 + q * 32;
      const uint32_t t0 = tmem_base + (uint32_t(q * 32) << 16) + acc * PBN;
#pragma unroll 1
      for (int c = half * NC; c < half * NC + NC; ++c) {
        uint32_t r[32];
        ptx::tmem_ld32(t0 + c * 32, r);
        const int col0 = nb * PBN + c * 32;
        if constexpr (TO) {
          uint4 auxc[4];
          if constexpr (AUX) {  // this lane's row of the staged residual chunk
            if (c == half * NC) ptx::mbar_wait(&auxbar[warp - 4], (aux_it - 1) & 1);
            const uint8_t* ab = stg + C::kAuxOff + (c - half * NC) * 2048;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              auxc[k] = *reinterpret_cast<const uint4*>(ab + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4));
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) auxc[k] = auxn[k], auxn[k] = auxn2[k];
            if (c + 2 < half * NC + NC) aux_row_prefetch<EPI>(ep, row0 + lane, col0 + 64, M, N, auxn2);
          }
          const uint32_t biasc = biasn;
          if (c + 1 < half * NC + NC) biasn = bias_prefetch(ep, col0 + 32, N, lane);
          ptx::tmem_ld_wait();
          // stream-K fix-up: + the partial tiles (loads issued here, not a chunk ahead: the
          // prefetch registers pushed the GELU'-epilogue instantiation into local-memory
          // spills and cost it 30 % in the step, profiles/r02bq_launch_summary_cfg3_b2.txt)
          for (int pq = q_lo; pq < pair; ++pq) {
            const float* pc = slot_of(pq) + size_t((q * 2 + half) * NC + (c - half * NC)) * 32 * 32;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 v = *reinterpret_cast<const float4*>(pc + (k * 32 + lane) * 4);
              r[4 * k] = __float_as_uint(__uint_as_float(r[4 * k]) + v.x);
              r[4 * k + 1] = __float_as_uint(__uint_as_float(r[4 * k + 1]) + v.y);
              r[4 * k + 2] = __float_as_uint(__uint_as_float(r[4 * k + 2]) + v.z);
              r[4 * k + 3] = __float_as_uint(__uint_as_float(r[4 * k + 3]) + v.w);
            }
          }
          if (row0 < M && col0 < N)
            epilogue_chunk_tma<EPI>(ep, &to, &to2, row0, col0, r, stg, lane, nbuf, auxc, biasc);
        } else {
          EpiPre cur = pre;
          if (c + 1 < half * NC + NC)
            epilogue_prefetch<EPI>(ep, row0, col0 + 32, M, N, lane, (ksplit > 1 || sk || ep.atomic_acc), pre);
          ptx::tmem_ld_wait();
          if (row0 < M && col0 < N)
            epilogue_chunk<EPI>(ep, row0, col0, M, N, r, stg, lane, (ksplit > 1 || sk || ep.atomic_acc), cur);
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      GEMM_TRACE(warp == 4 && lane == 0, it, 3);
      GEMM_TRACE(warp == 11 && lane == 0, it, 5);
      if (lane == 0) ptx::mbar_arrive_leader_relaxed(&tempty[acc]);
      if (itm.fixup) {  // every epilogue warp of this CTA has read the partials: re-arm
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kPairEpiWarps) : "memory");
        if (warp == 4 && lane == 0)
          for (int pq = q_lo; pq < pair; ++pq) flags[pq * 2 + int(cta)] = 0;
      }
    }
    if constexpr (TO)
      if (lane == 0) ptx::bulk_wait0();  // the bulk stores / reduces have completed
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem_base, C::kTmemCols);
  }
}

// Whether a launch takes the TMA-store epilogue, and its output tensor maps: every epilogue
// but kStoreF32, when the output rows (and the aux / out2 operands) are 16-byte aligned and
// N is whole 32-column chunks (CK_GEMM_TMA_OUT=0: the register epilogue everywhere; =1:
// not for bias+residual).
template <int EPI>
bool tma_out(const EpiArgs& ep, int M, int N, CUtensorMap& to, CUtensorMap& to2) {
  static const int tma_out_mode = [] {  // 0 off, 1 stores + accumulates, 2 also bias+residual
    const char* e = std::getenv("CK_GEMM_TMA_OUT");
    return e ? atoi(e) : 2;
  }();
  const bool tma_out_on = tma_out_mode >= (EPI == kBiasResid ? 2 : 1);
  constexpr bool kTmaCapable = EPI != kStoreF32;
  constexpr int esz = EPI == kAccF32 ? 4 : 2;
  const bool use_tma = kTmaCapable && tma_out_on && (reinterpret_cast<uintptr_t>(ep.out) % 16) == 0 &&
                       (ep.ldo * esz) % 16 == 0 && (!ep.bias || (reinterpret_cast<uintptr_t>(ep.bias) % 16) == 0) &&
                       ((EPI != kBiasResid && EPI != kGeluBwd) ||
                        ((reinterpret_cast<uintptr_t>(ep.aux) % 16) == 0 && ep.ld_aux % 8 == 0)) &&
                       (EPI != kBiasGelu || ((reinterpret_cast<uintptr_t>(ep.out2) % 16) == 0 && ep.ld_out2 % 8 == 0)) &&
                       (N % 32) == 0 && M >= 32;
  if (!use_tma) return false;
  to = EPI == kAccF32 ? cuda::make_map_2d_f32(ep.out, N, M, ep.ldo, 32, 32)
                      : cuda::make_map_2d_bf16(ep.out, N, M, ep.ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
  to2 = EPI == kBiasGelu ? cuda::make_map_2d_bf16(ep.out2, N, M, ep.ld_out2, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B) : to;
  return true;
}

// Stream-K (the CTA-pair kernel's WorkList) pays when whole 256 x PBN tiles leave many
// pairs idle in the last wave (efficiency tiles / (waves * pairs) < 0.85) and every pair
// gets a few K-blocks.  bf16 epilogues need the caller's workspace for the fp32 partial
// tiles (one 256 x PBN slot per pair) + the completion counters; fp32 accumulate needs
// none.  CK_GEMM_STREAMK=0 disables it.
//
// Measured (graph-timed, profiles/r02x_*, r02z_*): for the fp32 accumulate of the weight
// gradients with more tiles than pairs (75 / 100 tiles on 74 pairs) it beats whole tiles
// and two K-slices by 3-16 %; with fewer tiles than pairs two K-slices (split_k) stay
// better.  For the bf16 epilogues the fix-up -- a 128 KB fp32 partial per CTA written and
// read back through L2 before the epilogue -- costs more than the idle pairs it fills
// (e.g. 2528 x 1280 x 1280: 17.8 vs 12.1 us), so it is only taken with CK_GEMM_STREAMK=2.
inline bool stream_k_ok(int epi, const EpiArgs& ep, int base, int slots, int K, int pbn) {
  static const int mode = [] {  // 0 off, 1 fp32 accumulate only (default), 2 also bf16
    const char* e = std::getenv("CK_GEMM_STREAMK");
    return e ? atoi(e) : 1;
  }();
  if (mode == 0 || epi == kStoreF32 || ep.ksplit > 0) return false;
  const int waves = (base + slots - 1) / slots;
  if (double(base) / double(waves * slots) >= 0.85) return false;
  const long long kb = (K + BK - 1) / BK;
  if (kb * base / slots < 8) return false;
  if (epi == kAccF32) return base >= slots;
  return mode >= 2 && ep.ws && ep.ws_elems >= (long long)slots * 2 * 128 * pbn + kSkFlagInts &&
         (reinterpret_cast<uintptr_t>(ep.ws) % 16) == 0;
}

template <int PBN, bool A_MN, bool B_MN, int EPI>
void launch_pair(int M, int N, int K, const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B,
                 long long ldb, const EpiArgs& ep, cudaStream_t st) {
  using C = PairCfg<PBN>;
  const CUtensorMap ta = A_MN ? cuda::make_map_2d_bf16(A, M, K, lda, 64, BK)
                              : cuda::make_map_2d_bf16(A, K, M, lda, 64, 128);
  const CUtensorMap tb = B_MN ? cuda::make_map_2d_bf16(B, N, K, ldb, 64, BK)
                              : cuda::make_map_2d_bf16(B, K, N, ldb, 64, PBN / 2);
  const int base = ((M + 255) / 256) * ((N + PBN - 1) / PBN);
  const int slots = cuda::num_sms() / 2;
  int ks = split_k(EPI, base, slots, K, ep.ksplit);
  int tiles = base * ks;
  int pairs = tiles < slots ? tiles : slots;
  CUtensorMap to, to2;
  if constexpr (EPI != kStoreF32) {
    if (tma_out<EPI>(ep, M, N, to, to2)) {
      // stream-K when whole tiles would leave >= 15 % of the pairs idle in the last wave
      const int sk = stream_k_ok(EPI, ep, base, slots, K, PBN) ? 1 : 0;
      if (sk) ks = 1, tiles = base, pairs = slots;
      using CT = PairCfg<PBN, EPI == kBiasResid>;
      if constexpr (EPI == kBiasResid)  // the residual, in the output's 32 x 32 swizzled chunk layout
        to2 = cuda::make_map_2d_bf16(ep.aux, N, M, ep.ld_aux, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
      auto kern = k_gemm2<PBN, A_MN, B_MN, EPI, true>;
      static bool attr = false;
      if (!attr) {
        CK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, CT::kSmem));
        attr = true;
      }
      cuda::launch(kern, dim3(2 * pairs), dim3(128 + 32 * kPairEpiWarps), CT::kSmem, st, ta, tb, to, to2, ep, M, N,
                   K, ks, sk);
      CK_CUDA(cudaGetLastError());
      return;
    }
  }
  auto kern = k_gemm2<PBN, A_MN, B_MN, EPI, false>;
  static bool attr = false;
  if (!attr) {
    CK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr = true;
  }
  cuda::launch(kern, dim3(2 * pairs), dim3(128 + 32 * kPairEpiWarps), C::kSmem, st, ta, tb, ta, ta, ep, M, N, K, ks,
               0);
  CK_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void launch(int M, int N, int K, const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B,
            long long ldb, const EpiArgs& ep, cudaStream_t st) {
  using C = Cfg<BN>;
  const CUtensorMap ta = A_MN ? cuda::make_map_2d_bf16(A, M, K, lda, 64, BK)
                              : cuda::make_map_2d_bf16(A, K, M, lda, 64, BM);
  const CUtensorMap tb = B_MN ? cuda::make_map_2d_bf16(B, N, K, ldb, 64, BK)
                              : cuda::make_map_2d_bf16(B, K, N, ldb, 64, BN);
  const int base = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int ks = split_k(EPI, base, cuda::num_sms(), K, ep.ksplit);
  const int tiles = base * ks;
  const int grid = tiles < cuda::num_sms() ? tiles : cuda::num_sms();
  CUtensorMap to, to2;
  if constexpr (EPI != kStoreF32) {
    if (tma_out<EPI>(ep, M, N, to, to2)) {
      auto kern = k_gemm<BN, A_MN, B_MN, EPI, true>;
      static bool attr = false;
      if (!attr) {
        CK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
        attr = true;
      }
      cuda::launch(kern, dim3(grid), dim3(256), C::kSmem, st, ta, tb, to, to2, ep, M, N, K, ks);
      CK_CUDA(cudaGetLastError());
      return;
    }
  }
  auto kern = k_gemm<BN, A_MN, B_MN, EPI, false>;
  static bool attr = false;  // one-time per instantiation
  if (!attr) {
    CK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    attr = true;
  }
  cuda::launch(kern, dim3(grid), dim3(256), C::kSmem, st, ta, tb, ta, ta, ep, M, N, K, ks);
  CK_CUDA(cudaGetLastError());
}

template <int BN, bool A_MN, bool B_MN, int EPI>
void launch_any(int M, int N, int K, const __nv_bfloat16* A, long long lda, const __nv_bfloat16* B,
                long long ldb, const EpiArgs& ep, cudaStream_t st) {
  if constexpr (BN == 0) launch_pair<256, A_MN, B_MN, EPI>(M, N, K, A, lda, B, ldb, ep, st);
  else if constexpr (BN == 1 && !B_MN) launch_pair<192, A_MN, B_MN, EPI>(M, N, K, A, lda, B, ldb, ep, st);
  else if constexpr (BN == 1) launch_pair<256, A_MN, B_MN, EPI>(M, N, K, A, lda, B, ldb, ep, st);  // K-major B only
  else launch<BN, A_MN, B_MN, EPI>(M, N, K, A, lda, B, ldb, ep, st);
}

template <int BN, bool A_MN, bool B_MN>
void by_epi(Epi epi, int M, int N, int K, const __nv_bfloat16* A, long long lda,
            const __nv_bfloat16* B, long long ldb, const EpiArgs& ep, cudaStream_t st) {
  switch (epi) {
    case kStoreBF16: return launch_any<BN, A_MN, B_MN, kStoreBF16>(M, N, K, A, lda, B, ldb, ep, st);
    case kStoreF32: return launch_any<BN, A_MN, B_MN, kStoreF32>(M, N, K, A, lda, B, ldb, ep, st);
    case kAccF32: return launch_any<BN, A_MN, B_MN, kAccF32>(M, N, K, A, lda, B, ldb, ep, st);
    default: break;
  }
  if constexpr (!A_MN && !B_MN) {
    if (epi == kBiasGelu) return launch_any<BN, false, false, kBiasGelu>(M, N, K, A, lda, B, ldb, ep, st);
    if (epi == kBiasResid) return launch_any<BN, false, false, kBiasResid>(M, N, K, A, lda, B, ldb, ep, st);
  }
  if constexpr (!A_MN && B_MN) {
    if (epi == kGeluBwd) return launch_any<BN, false, true, kGeluBwd>(M, N, K, A, lda, B, ldb, ep, st);
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

// Tile configuration by a wave model calibrated on B200 (scripts/gemm_tile_sweep.py):
// time = waves x per-tile work / per-slot rate, waves over the slots the configuration
// keeps resident (74 CTA pairs or 148 CTAs), split-K included for the fp32 accumulate.
// Per-slot rates (TFLOP/s): CTA pair 256x256 24.6, 128x256 11.4, 128x128 7.0, 128x64 3.6
// -- the narrow tiles are operand-bound but put more SMs on problems with few output
// tiles and a deep K (the small-M stage shapes of GPT-2 1.3B / Bert-48).
// With a split-K workspace the bf16 epilogues may also be cut into 2-4 K-slices (each
// >= 8 K-blocks deep); that variant pays the finalize pass: a launch plus M*N*(8+2)
// bytes (+2 residual / gelu operand, +2 second output) at ~4 TB/s, and a per-wave
// fixed cost for the shallower tiles.
// Per-pair TFLOP/s of the 256 x 192 tile in the wave model (CK_GEMM_RATE192, e.g. 23).
// Off by default: timed alone it is 6-8 % faster on the N = 1280 shapes (50 -> 70 busy
// pairs), but in the one-GPU step, where eight ranks' kernels share the SMs, the idle
// pairs of a 256-wide launch are used by the other ranks anyway and the narrower tile's
// lower work per SM (operand feed) cost 3.6 % of throughput (profiles/r02ax_*).
inline double rate192() {
  static const double r = [] {
    const char* e = std::getenv("CK_GEMM_RATE192");
    return e ? atof(e) : 0.0;
  }();
  return r;
}
// CTA pair 256 x 192 (K-major B only: an MN-major B half of 96 rows is not whole 64-row
// swizzle atoms): three quarters of the pair tile's work per output tile, for the N = 1280
// shapes of GPT-2 1.3B where 256-wide tiles fill 50 of 74 pairs (70 with 192 columns).
struct TilePlan {
  int choice;  // 0 = CTA pair 256x256, 1 = CTA pair 256x192, else single-CTA 128 x choice
  int ks;      // K-slices (bf16 epilogues through the workspace when > 1)
};

TilePlan pick_tile(Epi epi, int M, int N, int K, bool can_split, bool b_mn) {
  struct Cand {
    int choice, bm, bn, slots;
    double rate;
  };
  const Cand cands[] = {{0, 256, 256, cuda::num_sms() / 2, 24.6}, {1, 256, 192, cuda::num_sms() / 2, rate192()},
                        {256, BM, 256, cuda::num_sms(), 11.4}, {128, BM, 128, cuda::num_sms(), 7.0},
                        {64, BM, 64, cuda::num_sms(), 3.6}};
  const int kb = (K + BK - 1) / BK;
  const int kmax = can_split ? std::max(1, std::min(4, kb / 8)) : 1;
  const double wave_fixed = 1.5e6;  // ps: prologue / fill / exposed epilogue per wave
  const double fin = 2.5e6 + double(M) * N * (10.0 + (epi == kBiasResid || epi == kGeluBwd || epi == kBiasGelu ? 2.0 : 0.0)) /
                                 4.0e12 * 1e12;
  TilePlan best{128, 1};
  double best_t = 1e300;
  for (const Cand& c : cands) {
    if (c.choice == 0 && (M < 256 || N < 256)) continue;
    if (c.choice == 1 && (M < 256 || N < 192 || b_mn || c.rate <= 0.0)) continue;
    if (c.choice == 256 && N <= 128) continue;
    const long long tiles = (long long)((M + c.bm - 1) / c.bm) * ((N + c.bn - 1) / c.bn);
    for (int kq = 1; kq <= (epi == kAccF32 ? 1 : kmax); ++kq) {
      const int ks = epi == kAccF32 ? split_k(epi, int(std::min<long long>(tiles, 1 << 30)), c.slots, K) : kq;
      const long long units = tiles * ks, waves = (units + c.slots - 1) / c.slots;
      const double kdepth = double((K + ks - 1) / ks);
      double t = double(waves) * (2.0 * c.bm * c.bn * kdepth) / c.rate;
      if (epi != kAccF32 && ks > 1) t += double(waves) * wave_fixed + fin;
      if (t < best_t * 0.98) best_t = t, best = {c.choice, epi == kAccF32 ? 0 : ks};  // prefer earlier (larger) on near-ties
    }
  }
  return best;
}

int pick_tile(Epi epi, int M, int N, int K) { return pick_tile(epi, M, N, K, false, false).choice; }

namespace {

void dispatch(int choice, Epi epi, bool a_mn, bool b_mn, int M, int N, int K, const __nv_bfloat16* A, long long lda,
              const __nv_bfloat16* B, long long ldb, const EpiArgs& ep, cudaStream_t st) {
  if ((choice == 0 && (M < 256 || N < 256)) || (choice == 1 && (M < 256 || N < 192))) choice = 128;
  if (choice == 0) by_layout<0>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
  else if (choice == 1) by_layout<1>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
  else if (choice == 256) by_layout<256>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
  else if (choice == 64) by_layout<64>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
  else by_layout<128>(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, ep, st);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) % 16) == 0; }

// The workspace route needs whole 8-column groups and 16-byte aligned operands.
bool split_ok(Epi epi, int M, int N, const EpiArgs& ep) {
  if (!ep.ws || epi == kAccF32 || epi == kStoreF32 || ep.ws_elems < (long long)M * N) return false;
  if (N % 8 || ep.ldo % 8 || !aligned16(ep.out) || !aligned16(ep.ws)) return false;
  if (ep.bias && !aligned16(ep.bias)) return false;
  if ((epi == kBiasResid || epi == kGeluBwd) && (!ep.aux || ep.ld_aux % 8 || !aligned16(ep.aux))) return false;
  if (epi == kBiasGelu && (!ep.out2 || ep.ld_out2 % 8 || !aligned16(ep.out2))) return false;
  if (epi == kGeluBwd && ep.colsum && !aligned16(ep.colsum)) return false;
  return true;
}

template <int EPI>
void finalize(const EpiArgs& ep, int M, int N, cudaStream_t st) {
  const dim3 grid((N / 8 + 127) / 128, (M + kFinRows - 1) / kFinRows);
  cuda::launch(k_splitk_finalize<EPI>, grid, dim3(128), 0, st, ep.ws, ep, M, N);
  CK_CUDA(cudaGetLastError());
}

}  // namespace

void gemm(Epi epi, bool a_mn, bool b_mn, int M, int N, int K, const __nv_bfloat16* A, long long lda,
          const __nv_bfloat16* B, long long ldb, const EpiArgs& ep, cudaStream_t st) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  if ((lda % 8) || (ldb % 8) || (reinterpret_cast<uintptr_t>(A) % 16) || (reinterpret_cast<uintptr_t>(B) % 16))
    throw chimera::capi::InternalError("gemm: operands must be 16-byte aligned with ld % 8 == 0");
  // CTA-pair 256 x 256 or single-CTA 128 x {256, 128, 64} tiles, split-K slices (pick_tile).
  static const int force = [] {
    const char* e = std::getenv("CK_GEMM_TILE");  // "pair" | "pair192" | "256" | "128" | "64" (benchmarks)
    if (!e) return -1;
    const std::string v(e);
    return v == "pair" ? 0 : v == "pair192" ? 1 : v == "256" ? 256 : v == "64" ? 64 : 128;
  }();
  // The workspace route is OFF unless CK_GEMM_SPLIT_BF16=1 (wave model decides) or n > 1
  // (n slices), or a caller forces a slice count: graph-timed on B200 it never beat the
  // best unsplit tile on the 632 / 1264 / 2528-row stage shapes -- the fp32 partial
  // reduce-adds plus the finalize pass cost more than the wave they fill
  // (profiles/r02f_gemm_split_sweep.jsonl).
  static const int force_split = [] {
    const char* e = std::getenv("CK_GEMM_SPLIT_BF16");
    return e ? atoi(e) : 0;
  }();
  const bool can_split = (force_split != 0 || ep.ksplit >= 1) && split_ok(epi, M, N, ep);
  TilePlan plan = pick_tile(epi, M, N, K, can_split, b_mn);
  if (force >= 0) plan.choice = force;
  if (ep.tile >= 0) plan.choice = ep.tile;
  if (can_split && force_split > 1) plan.ks = force_split;
  if (can_split && ep.ksplit >= 1) plan.ks = ep.ksplit;  // caller-forced (tests / benchmarks); 1 = no split
  if (plan.ks > 1 && can_split) {  // K-slices into the workspace, then the epilogue pass
    EpiArgs part;
    part.out = ep.ws;
    part.ldo = N;
    part.atomic_acc = true;
    part.ksplit = plan.ks;
    dispatch(plan.choice, kAccF32, a_mn, b_mn, M, N, K, A, lda, B, ldb, part, st);
    switch (epi) {
      case kStoreBF16: return finalize<kStoreBF16>(ep, M, N, st);
      case kBiasGelu: return finalize<kBiasGelu>(ep, M, N, st);
      case kBiasResid: return finalize<kBiasResid>(ep, M, N, st);
      case kGeluBwd: return finalize<kGeluBwd>(ep, M, N, st);
      default: break;
    }
    throw chimera::capi::InternalError("gemm: split-K epilogue not supported");
  }
  EpiArgs e2 = ep;
  e2.ksplit = epi == kAccF32 ? ep.ksplit : 0;  // fp32 accumulate: a caller-forced slice count stands
  dispatch(plan.choice, epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, e2, st);
}

}  // namespace chimera::gemm

extern "C" {

// Test / integration entry: all pointers are device pointers; stream may be 0.
CK_API int ck_gemm_bf16_ex(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A,
                           long long lda, const void* B, long long ldb, void* out, long long ldo,
                           const void* bias, const void* aux, long long ld_aux, void* out2,
                           long long ld_out2, float* colsum, void* stream) {
  return chimera::capi::guarded([&] {
    chimera::gemm::EpiArgs ep;
    ep.out = out;
    ep.ldo = ldo;
    ep.bias = static_cast<const __nv_bfloat16*>(bias);
    ep.aux = static_cast<const __nv_bfloat16*>(aux);
    ep.ld_aux = ld_aux;
    ep.out2 = static_cast<__nv_bfloat16*>(out2);
    ep.ld_out2 = ld_out2;
    ep.colsum = colsum;
    chimera::gemm::gemm(static_cast<chimera::gemm::Epi>(epi), a_mn != 0, b_mn != 0, M, N, K,
                        static_cast<const __nv_bfloat16*>(A), lda, static_cast<const __nv_bfloat16*>(B),
                        ldb, ep, static_cast<cudaStream_t>(stream));
  });
}

// ck_gemm_bf16_ex with a split-K workspace (fp32, zero-filled, >= M*N; left zeroed):
// ksplit > 1 forces that many K-slices for a bf16 epilogue, 0 lets the wave model choose.
CK_API int ck_gemm_bf16_split(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A, long long lda,
                              const void* B, long long ldb, void* out, long long ldo, const void* bias,
                              const void* aux, long long ld_aux, void* out2, long long ld_out2, float* colsum,
                              float* ws, long long ws_elems, int ksplit, int tile, void* stream) {
  return chimera::capi::guarded([&] {
    chimera::gemm::EpiArgs ep;
    ep.out = out;
    ep.ldo = ldo;
    ep.bias = static_cast<const __nv_bfloat16*>(bias);
    ep.aux = static_cast<const __nv_bfloat16*>(aux);
    ep.ld_aux = ld_aux;
    ep.out2 = static_cast<__nv_bfloat16*>(out2);
    ep.ld_out2 = ld_out2;
    ep.colsum = colsum;
    ep.ws = ws;
    ep.ws_elems = ws_elems;
    ep.ksplit = ksplit;  // honoured by gemm() as the forced slice count when > 1
    ep.tile = tile;
    chimera::gemm::gemm(static_cast<chimera::gemm::Epi>(epi), a_mn != 0, b_mn != 0, M, N, K,
                        static_cast<const __nv_bfloat16*>(A), lda, static_cast<const __nv_bfloat16*>(B),
                        ldb, ep, static_cast<cudaStream_t>(stream));
  });
}

CK_API int ck_gemm_bf16(int epi, int a_mn, int b_mn, int M, int N, int K, const void* A,
                        long long lda, const void* B, long long ldb, void* out, long long ldo,
                        const void* bias, const void* aux, long long ld_aux, void* out2,
                        long long ld_out2, void* stream) {
  return ck_gemm_bf16_ex(epi, a_mn, b_mn, M, N, K, A, lda, B, ldb, out, ldo, bias, aux, ld_aux, out2, ld_out2,
                         nullptr, stream);
}

}  // extern "C"
