// Flash attention (head dim 64) forward and backward over the packed qkv buffer the
// QKV GEMM writes, so no head split / transpose kernel runs between them.
//
// Forward: CTA = (64-query block, batch*head), 4 warps x 16 query rows; K/V 64-key
// blocks double-buffered in shared memory with cp.async; S = Q K^T and O += P V on
// the bf16 tensor pipe (mma.sync m16n8k16, fp32 accumulate), online softmax in the
// exp2 domain; the log-sum-exp per row is kept for the backward pass.
// Backward: CTA = (64-key block, batch*head), 4 warps x 16 keys; for every query block
// recompute P^T = exp(S^T - lse), dV += P^T dO, dP^T = V dO^T, dS^T = P^T (dP^T - D),
// dK += dS^T Q (registers), dQ += dS K (fp32 atomics into a scratch accumulator).
// Causal masking (GPT-2) skips key blocks beyond the diagonal; sequence tails are
// masked (seq need not be a multiple of 64, e.g. 632).
//
// These run on the legacy mma.sync tensor path (HMMA); a tcgen05/TMEM version is the
// planned upgrade, attention being ~15% of the GPT-2 stage FLOPs.
#include "chimera_ck.h"
#include "common.cuh"
#include "ops.cuh"

namespace chimera::ops {

namespace {

constexpr int kTile = 64, kHd = 64, kLd = 72;  // smem row stride (elements), conflict-free
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const bf16* p) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(s));
}
__device__ __forceinline__ uint32_t ld32(const bf16* p) { return *reinterpret_cast<const uint32_t*>(p); }
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 64 rows x 64 columns of bf16 from a row-strided global matrix into smem (stride kLd).
__device__ __forceinline__ void load_tile(bf16* s, const bf16* g, long long ld, int row0, int rows) {
  for (int c = threadIdx.x; c < kTile * 8; c += blockDim.x) {
    const int r = c >> 3, ch = c & 7;
    const bool ok = row0 + r < rows;
    cp_async16(s + r * kLd + ch * 8, g + (long long)(ok ? row0 + r : 0) * ld + ch * 8, ok);
  }
}

// A fragments (16 rows x 64 cols) of a row-major smem tile: a[kc] covers cols kc*16..+15.
__device__ __forceinline__ void load_a_frags(uint32_t (&a)[4][4], const bf16* s, int row0) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    const bf16* p = s + (row0 + g) * kLd + kc * 16 + 2 * t;
    a[kc][0] = ld32(p);
    a[kc][1] = ld32(p + 8 * kLd);
    a[kc][2] = ld32(p + 8);
    a[kc][3] = ld32(p + 8 * kLd + 8);
  }
}

// acc[n] (16 x 8 tile n) += A (16 x 64) * B^T where B rows (= output columns) live
// row-major in smem: B(n-row, k) = s[(n*8 + g) * kLd + k].
__device__ __forceinline__ void mma_abt(float (&acc)[8][4], const uint32_t (&a)[4][4], const bf16* s) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
      const bf16* p = s + (n * 8 + g) * kLd + kc * 16 + 2 * t;
      mma16816(acc[n], a[kc], ld32(p), ld32(p + 8));
    }
}

// acc (16 x 64) += P (16 x 64, C-fragment layout in p[8][4]) * S where S is a
// row-major 64 x 64 smem tile (rows = reduction index).
__device__ __forceinline__ void mma_pv(float (&acc)[8][4], const float (&p)[8][4], const bf16* s) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    const uint32_t a[4] = {pack(p[2 * kc][0], p[2 * kc][1]), pack(p[2 * kc][2], p[2 * kc][3]),
                           pack(p[2 * kc + 1][0], p[2 * kc + 1][1]), pack(p[2 * kc + 1][2], p[2 * kc + 1][3])};
#pragma unroll
    for (int dn = 0; dn < 8; dn += 2) {
      uint32_t r[4];
      ldsm_x4_t(r, s + (kc * 16 + (lane & 7) + 8 * ((lane >> 3) & 1)) * kLd + dn * 8 + 8 * (lane >> 4));
      mma16816(acc[dn], a, r[0], r[1]);
      mma16816(acc[dn + 1], a, r[2], r[3]);
    }
  }
}

template <bool CAUSAL>
__global__ void __launch_bounds__(128) k_attn_fwd(const bf16* __restrict__ qkv, bf16* __restrict__ out,
                                                  float* __restrict__ lse, int seq, int H) {
  __shared__ alignas(128) bf16 sQ[kTile * kLd];
  __shared__ alignas(128) bf16 sK[2][kTile * kLd];
  __shared__ alignas(128) bf16 sV[2][kTile * kLd];
  const int qb = blockIdx.x, bh = blockIdx.y, b = bh / H, hd = bh % H;
  const long long ld = 3LL * H * kHd;
  const bf16* base = qkv + (long long)b * seq * ld;
  const bf16* gq = base + hd * kHd;
  const bf16* gk = base + (long long)H * kHd + hd * kHd;
  const bf16* gv = base + 2LL * H * kHd + hd * kHd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float sl2 = 0.125f * kLog2e;  // softmax scale 1/sqrt(64), exp2 domain

  const int nkb = CAUSAL ? qb + 1 : (seq + kTile - 1) / kTile;
  load_tile(sQ, gq, ld, qb * kTile, seq);
  load_tile(sK[0], gk, ld, 0, seq);
  load_tile(sV[0], gv, ld, 0, seq);
  cp_commit();

  uint32_t qa[4][4];
  float o[8][4] = {};
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  const int qrow0 = qb * kTile + warp * 16 + g;

  for (int kb = 0; kb < nkb; ++kb) {
    const int st = kb & 1;
    if (kb + 1 < nkb) {
      load_tile(sK[st ^ 1], gk, ld, (kb + 1) * kTile, seq);
      load_tile(sV[st ^ 1], gv, ld, (kb + 1) * kTile, seq);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (kb == 0) load_a_frags(qa, sQ, warp * 16);

    float s[8][4] = {};
    mma_abt(s, qa, sK[st]);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int key = kb * kTile + n * 8 + 2 * t + (j & 1);
        const int q = qrow0 + 8 * (j >> 1);
        float v = s[n][j] * sl2;
        if (key >= seq || (CAUSAL && key > q)) v = -INFINITY;
        s[n][j] = v;
        mx[j >> 1] = fmaxf(mx[j >> 1], v);
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m[r], mx[r]);
      const float safe = mn == -INFINITY ? 0.f : mn;
      const float alpha = exp2f(m[r] - safe);
      m[r] = mn;
      l[r] *= alpha;
#pragma unroll
      for (int dn = 0; dn < 8; ++dn) o[dn][2 * r] *= alpha, o[dn][2 * r + 1] *= alpha;
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const float p0 = exp2f(s[n][2 * r] - safe), p1 = exp2f(s[n][2 * r + 1] - safe);
        s[n][2 * r] = p0, s[n][2 * r + 1] = p1;
        l[r] += p0 + p1;
      }
    }
    mma_pv(o, s, sV[st]);
    __syncthreads();
  }

#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
    const int q = qrow0 + 8 * r;
    if (q >= seq) continue;
    const float inv = l[r] > 0.f ? 1.f / l[r] : 0.f;
    bf16* orow = out + ((long long)b * seq + q) * (H * kHd) + hd * kHd;
#pragma unroll
    for (int dn = 0; dn < 8; ++dn)
      *reinterpret_cast<uint32_t*>(orow + dn * 8 + 2 * t) = pack(o[dn][2 * r] * inv, o[dn][2 * r + 1] * inv);
    if (t == 0) lse[(long long)bh * seq + q] = (m[r] + __log2f(l[r])) / kLog2e;
  }
}

// D[bh][q] = sum_d dO[q][d] * O[q][d]: 8 threads per (token, head) row, 16-byte loads,
// two rows per thread in flight (pure HBM stream: 2 x M*H*128 bytes).  With `dq` set, the
// same threads also zero the fp32 dQ accumulator (M*H*64 floats, 32 bytes per row part).
__global__ void __launch_bounds__(256) k_attn_bwd_dot(const bf16* __restrict__ out, const bf16* __restrict__ dout,
                                                      float* __restrict__ D, float* __restrict__ dq, int M, int seq,
                                                      int H) {
  cuda::pdl_wait();
  const long long rows = (long long)M * H;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int part = threadIdx.x & 7;
  const long long stride = (long long)gridDim.x * blockDim.x / 8;
  for (long long r0 = t >> 3; r0 < rows; r0 += 2 * stride) {
    if (dq) {  // row r of [tok][H*64] is the contiguous 64 floats at r*64
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      float4* p0 = reinterpret_cast<float4*>(dq + r0 * kHd + part * 8);
      p0[0] = z;
      p0[1] = z;
      if (r0 + stride < rows) {
        float4* p1 = reinterpret_cast<float4*>(dq + (r0 + stride) * kHd + part * 8);
        p1[0] = z;
        p1[1] = z;
      }
    }
    const long long r1 = r0 + stride;
    uint4 a0 = __ldcs(reinterpret_cast<const uint4*>(out + r0 * kHd + part * 8));
    uint4 c0 = __ldcs(reinterpret_cast<const uint4*>(dout + r0 * kHd + part * 8));
    uint4 a1 = make_uint4(0, 0, 0, 0), c1 = a1;
    if (r1 < rows) {
      a1 = __ldcs(reinterpret_cast<const uint4*>(out + r1 * kHd + part * 8));
      c1 = __ldcs(reinterpret_cast<const uint4*>(dout + r1 * kHd + part * 8));
    }
    auto dot8 = [](uint4 a, uint4 c) {
      const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(&c);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 u = __bfloat1622float2(x[i]), v = __bfloat1622float2(y[i]);
        s = fmaf(u.x, v.x, fmaf(u.y, v.y, s));
      }
      return s;
    };
    float s0 = dot8(a0, c0), s1 = dot8(a1, c1);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (part == 0) {
      // row r = tok * H + hd  ->  D[(b * H + hd) * seq + q]
      const int tok0 = int(r0 / H), hd0 = int(r0 % H);
      D[((long long)(tok0 / seq) * H + hd0) * seq + tok0 % seq] = s0;
      if (r1 < rows) {
        const int tok1 = int(r1 / H), hd1 = int(r1 % H);
        D[((long long)(tok1 / seq) * H + hd1) * seq + tok1 % seq] = s1;
      }
    }
  }
}

template <bool CAUSAL>
__global__ void __launch_bounds__(128) k_attn_bwd(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                  const float* __restrict__ lse, const float* __restrict__ Dv,
                                                  float* __restrict__ dq_acc, bf16* __restrict__ dqkv, int seq,
                                                  int H) {
  __shared__ alignas(128) bf16 sK[kTile * kLd];
  __shared__ alignas(128) bf16 sV[kTile * kLd];
  __shared__ alignas(128) bf16 sQ[kTile * kLd];
  __shared__ alignas(128) bf16 sdO[kTile * kLd];
  __shared__ alignas(128) bf16 sdS[kTile * kLd];
  __shared__ float sL[kTile], sD[kTile];
  const int kb = blockIdx.x, bh = blockIdx.y, b = bh / H, hd = bh % H;  // causal: kb 0 has most work
  const long long ld = 3LL * H * kHd, ldo = (long long)H * kHd;
  const bf16* base = qkv + (long long)b * seq * ld;
  const bf16* gq = base + hd * kHd;
  const bf16* gk = base + (long long)H * kHd + hd * kHd;
  const bf16* gv = base + 2LL * H * kHd + hd * kHd;
  const bf16* gdo = dout + (long long)b * seq * ldo + hd * kHd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const float sl2 = 0.125f * kLog2e;

  load_tile(sK, gk, ld, kb * kTile, seq);
  load_tile(sV, gv, ld, kb * kTile, seq);
  cp_commit();
  cp_wait<0>();
  __syncthreads();
  uint32_t ka[4][4], va[4][4];
  load_a_frags(ka, sK, warp * 16);
  load_a_frags(va, sV, warp * 16);
  float dk[8][4] = {}, dv[8][4] = {};
  const int key0 = kb * kTile + warp * 16 + g;  // keys key0 and key0 + 8 for this thread
  const int nqb = (seq + kTile - 1) / kTile;

  for (int qb = CAUSAL ? kb : 0; qb < nqb; ++qb) {
    load_tile(sQ, gq, ld, qb * kTile, seq);
    load_tile(sdO, gdo, ldo, qb * kTile, seq);
    cp_commit();
    if (threadIdx.x < kTile) {
      const int q = qb * kTile + threadIdx.x;
      sL[threadIdx.x] = q < seq ? lse[(long long)bh * seq + q] * kLog2e : 0.f;
      sD[threadIdx.x] = q < seq ? Dv[(long long)bh * seq + q] : 0.f;
    }
    cp_wait<0>();
    __syncthreads();

    float p[8][4] = {}, dp[8][4] = {};
    mma_abt(p, ka, sQ);    // S^T (16 keys x 64 queries)
    mma_abt(dp, va, sdO);  // dP^T
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ql = n * 8 + 2 * t + (j & 1);
        const int q = qb * kTile + ql, key = key0 + 8 * (j >> 1);
        const bool keep = q < seq && key < seq && !(CAUSAL && key > q);
        const float pv = keep ? exp2f(p[n][j] * sl2 - sL[ql]) : 0.f;
        p[n][j] = pv;
        dp[n][j] = pv * (dp[n][j] - sD[ql]);  // dS^T (unscaled)
      }
    mma_pv(dv, p, sdO);  // dV += P^T dO
    mma_pv(dk, dp, sQ);  // dK += dS^T Q   (scaled at the end)
    // dS^T -> smem for the dQ product
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      bf16* r0 = sdS + (warp * 16 + g) * kLd + n * 8 + 2 * t;
      *reinterpret_cast<uint32_t*>(r0) = pack(dp[n][0], dp[n][1]);
      *reinterpret_cast<uint32_t*>(r0 + 8 * kLd) = pack(dp[n][2], dp[n][3]);
    }
    __syncthreads();
    // dQ (64 q x 64 d) += dS (q x 64 keys) K; warp w owns queries w*16..+15.
    {
      float dq[8][4] = {};
#pragma unroll
      for (int kc = 0; kc < 4; ++kc) {
        uint32_t a[4];
        // A(q, key) = dS^T[key][q]: transposed 8x8 loads of the stored dS^T tile
        ldsm_x4_t(a, sdS + (kc * 16 + (lane & 7) + 8 * (lane >> 4)) * kLd + warp * 16 + 8 * ((lane >> 3) & 1));
#pragma unroll
        for (int dn = 0; dn < 8; dn += 2) {
          uint32_t r[4];
          ldsm_x4_t(r, sK + (kc * 16 + (lane & 7) + 8 * ((lane >> 3) & 1)) * kLd + dn * 8 + 8 * (lane >> 4));
          mma16816(dq[dn], a, r[0], r[1]);
          mma16816(dq[dn + 1], a, r[2], r[3]);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = qb * kTile + warp * 16 + g + 8 * r;
        if (q >= seq) continue;
        float* acc = dq_acc + ((long long)b * seq + q) * (H * kHd) + hd * kHd;
#pragma unroll
        for (int dn = 0; dn < 8; ++dn)  // vector fp32 atomic (sm_90+): 2 columns per op
          atomicAdd(reinterpret_cast<float2*>(acc + dn * 8 + 2 * t), make_float2(dq[dn][2 * r], dq[dn][2 * r + 1]));
      }
    }
    __syncthreads();
  }
  // dK (scaled) and dV for this key block
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int key = key0 + 8 * r;
    if (key >= seq) continue;
    bf16* row = dqkv + ((long long)b * seq + key) * ld;
#pragma unroll
    for (int dn = 0; dn < 8; ++dn) {
      *reinterpret_cast<uint32_t*>(row + (long long)H * kHd + hd * kHd + dn * 8 + 2 * t) =
          pack(dk[dn][2 * r] * 0.125f, dk[dn][2 * r + 1] * 0.125f);
      *reinterpret_cast<uint32_t*>(row + 2LL * H * kHd + hd * kHd + dn * 8 + 2 * t) =
          pack(dv[dn][2 * r], dv[dn][2 * r + 1]);
    }
  }
}

// dqkv[:, q-part] = bf16(dq_acc * scale)
// dQ (fp32 accumulator, scaled by 1/sqrt(d)) -> bf16 Q-part of dqkv (L2-resident stream)
// dQ (fp32 accumulator, scaled by 1/sqrt(d) here) -> the Q columns of dqkv in bf16; with
// dbias, also the Q part of the QKV bias gradient: column sums of the bf16 values written.
// threadIdx.x + blockIdx.y * blockDim.x <-> 8-column group (w / 8 of them, at most 256
// per CTA: any head count), threadIdx.y <-> one of 4 rows in flight; CTAs stride over
// row quads.
constexpr int kDqGroups = 256;
// kDqUnroll rows per thread in flight: one CTA per SM holds ~512 threads, so one row's
// 32 bytes per thread left the SMs ~2 TB/s short of HBM on this pure stream
constexpr int kDqUnroll = 4;
__global__ void __launch_bounds__(1024) k_dq_out(const float* __restrict__ acc, bf16* __restrict__ dqkv, int n_rows,
                                                 int H, float* __restrict__ dbias) {
  cuda::pdl_wait();
  const int w = H * kHd, g = blockIdx.y * blockDim.x + threadIdx.x;  // w is a multiple of 64
  const bool live = g < w / 8;
  const int rs = gridDim.x * 4;  // row stride between a thread's rows
  float cs[8] = {};
  for (int r0 = blockIdx.x * 4 + threadIdx.y; live && r0 < n_rows; r0 += kDqUnroll * rs) {
    float4 a[kDqUnroll], b[kDqUnroll];
#pragma unroll
    for (int u = 0; u < kDqUnroll; ++u)
      if (r0 + u * rs < n_rows) {
        const float4* p = reinterpret_cast<const float4*>(acc + (long long)(r0 + u * rs) * w) + 2 * g;
        a[u] = __ldcs(p), b[u] = __ldcs(p + 1);
      }
#pragma unroll
    for (int u = 0; u < kDqUnroll; ++u) {
      const int r = r0 + u * rs;
      if (r >= n_rows) break;
      const uint4 q = make_uint4(pack(a[u].x * 0.125f, a[u].y * 0.125f), pack(a[u].z * 0.125f, a[u].w * 0.125f),
                                 pack(b[u].x * 0.125f, b[u].y * 0.125f), pack(b[u].z * 0.125f, b[u].w * 0.125f));
      *reinterpret_cast<uint4*>(dqkv + (long long)r * 3 * w + 8 * g) = q;
      if (dbias) {
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
        for (int t = 0; t < 8; ++t) cs[t] += __bfloat162float(h[t]);
      }
    }
  }
  if (dbias) {  // reduce the 4 row lanes in shared memory: one atomic set per CTA and column group
    __shared__ float red[4][8 * kDqGroups];
    const int l = threadIdx.x;
#pragma unroll
    for (int t = 0; t < 8; ++t) red[threadIdx.y][8 * l + t] = cs[t];
    __syncthreads();
    if (threadIdx.y == 0 && live) {
#pragma unroll
      for (int t = 0; t < 8; ++t) cs[t] = red[0][8 * l + t] + red[1][8 * l + t] + red[2][8 * l + t] + red[3][8 * l + t];
      atomicAdd(reinterpret_cast<float4*>(dbias + 8 * g), make_float4(cs[0], cs[1], cs[2], cs[3]));
      atomicAdd(reinterpret_cast<float4*>(dbias + 8 * g + 4), make_float4(cs[4], cs[5], cs[6], cs[7]));
    }
  }
}

}  // namespace

void attn_fwd(const bf16* qkv, bf16* out, float* lse, int B, int seq, int H, bool causal,
              cudaStream_t st) {
  const dim3 grid((seq + kTile - 1) / kTile, B * H);
  if (causal) k_attn_fwd<true><<<grid, 128, 0, st>>>(qkv, out, lse, seq, H);
  else k_attn_fwd<false><<<grid, 128, 0, st>>>(qkv, out, lse, seq, H);
  CK_CUDA(cudaGetLastError());
}

// D (B*H*seq floats), then the fp32 dQ accumulator at a 128-byte boundary (vector
// accesses and the TMA reduce-add need an aligned base for any B*H*seq)
size_t attn_dq_offset(int B, int seq, int H) { return (size_t(B) * H * seq + 31) / 32 * 32; }
size_t attn_bwd_scratch_floats(int B, int seq, int H) {
  return attn_dq_offset(B, seq, H) + size_t(B) * seq * H * kHd;
}

void attn_bwd_dot(const bf16* out, const bf16* dout, float* D, int M, int seq, int H, cudaStream_t st, float* dq_zero) {
  cuda::launch(k_attn_bwd_dot, dim3(std::min<long long>(cuda::ceil_div((long long)M * H * 8, 512), 148LL * 8)),
               dim3(256), 0, st, out, dout, D, dq_zero, M, seq, H);
  CK_CUDA(cudaGetLastError());
}

void attn_dq_out(const float* dq, bf16* dqkv, int M, int H, cudaStream_t st, float* dbias) {
  const int ng = H * kHd / 8;  // 8-column groups per row
  if (dbias && (reinterpret_cast<uintptr_t>(dbias) % 16))
    throw chimera::capi::InternalError("attention: the bias-gradient pointer must be 16-byte aligned");
  const int bx = std::min(ng, kDqGroups), by = (ng + bx - 1) / bx;
  // one CTA per SM (per column slab): the bias-gradient atomics are one set per CTA
  cuda::launch(k_dq_out, dim3(std::min((M + 3) / 4, cuda::num_sms()), by), dim3(bx, 4), 0, st, dq, dqkv, M, H,
               dbias);
  CK_CUDA(cudaGetLastError());
}

void attn_bwd(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, bf16* dqkv,
              float* scratch, int B, int seq, int H, bool causal, cudaStream_t st) {
  float* D = scratch;
  float* dq = scratch + attn_dq_offset(B, seq, H);
  const int M = B * seq;
  attn_bwd_dot(out, dout, D, M, seq, H, st, dq);
  const dim3 grid((seq + kTile - 1) / kTile, B * H);
  if (causal) k_attn_bwd<true><<<grid, 128, 0, st>>>(qkv, dout, lse, D, dq, dqkv, seq, H);
  else k_attn_bwd<false><<<grid, 128, 0, st>>>(qkv, dout, lse, D, dq, dqkv, seq, H);
  attn_dq_out(dq, dqkv, M, H, st, nullptr);
  CK_CUDA(cudaGetLastError());
}

}  // namespace chimera::ops

extern "C" {
using chimera::ops::bf16;
CK_API int ck_attn_fwd(const void* qkv, void* out, float* lse, int B, int seq, int H, int causal, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::attn_fwd((const bf16*)qkv, (bf16*)out, lse, B, seq, H, causal != 0, (cudaStream_t)st);
  });
}
CK_API int ck_attn_bwd(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                       float* scratch, int B, int seq, int H, int causal, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::attn_bwd((const bf16*)qkv, (const bf16*)out, (const bf16*)dout, lse, (bf16*)dqkv, scratch,
                           B, seq, H, causal != 0, (cudaStream_t)st);
  });
}
CK_API long long ck_attn_bwd_scratch_floats(int B, int seq, int H) {
  return (long long)chimera::ops::attn_bwd_scratch_floats(B, seq, H);
}
}
