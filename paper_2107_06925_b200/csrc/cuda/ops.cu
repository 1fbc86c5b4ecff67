// HBM-bound kernels of the transformer stage: LayerNorm fwd/bwd, embedding, softmax
// cross-entropy (fused forward + backward, in place), bias gradients, SGD update.
// Roofline: bytes moved / measured HBM bandwidth.  Design rules applied: 16-byte
// vector accesses, one warp per row for row-wise ops (statistics stay in registers:
// two-pass exact mean/variance with no re-read), column reductions accumulated in
// registers across many rows before one atomic per column per CTA.
#include "chimera_ck.h"
#include "common.cuh"
#include "ops.cuh"
#include "ptx_sm100.cuh"

namespace chimera::ops {

namespace {

using cuda::ceil_div;

struct Vec8 {  // 8 bf16 <-> 8 fp32
  float f[8];
  __device__ __forceinline__ void set(const uint4& q) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 v = __bfloat1622float2(h[t]);
      f[2 * t] = v.x, f[2 * t + 1] = v.y;
    }
  }
  __device__ __forceinline__ void load(const bf16* p) { set(*reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void store(bf16* p) const {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int t = 0; t < 4; ++t) h[t] = __floats2bfloat162_rn(f[2 * t], f[2 * t + 1]);
    *reinterpret_cast<uint4*>(p) = q;
  }
  __device__ __forceinline__ Vec8 rounded() const {  // the values store() writes
    Vec8 r;
#pragma unroll
    for (int t = 0; t < 8; ++t) r.f[t] = __bfloat162float(__float2bfloat16_rn(f[t]));
    return r;
  }
};

// ------------------------------------------------------------------ LayerNorm --
// One warp per row; lane owns VPL chunks of 8 columns: column = (c * 32 + lane) * 8.
template <int VPL>
__global__ void __launch_bounds__(256) k_ln_fwd(const bf16* __restrict__ x, const bf16* __restrict__ g,
                                                const bf16* __restrict__ b, bf16* __restrict__ y,
                                                float* __restrict__ mean, float* __restrict__ rstd, int M) {
  cuda::pdl_wait();
  constexpr int h = VPL * 256;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= M) return;
  const bf16* xr = x + (long long)row * h;
  Vec8 v[VPL];
  uint4 graw[VPL], braw[VPL];  // gamma / beta requested with the row (their latency overlaps it)
#pragma unroll
  for (int c = 0; c < VPL; ++c) {
    graw[c] = *reinterpret_cast<const uint4*>(g + (c * 32 + lane) * 8);
    braw[c] = *reinterpret_cast<const uint4*>(b + (c * 32 + lane) * 8);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < VPL; ++c) {
    v[c].load(xr + (c * 32 + lane) * 8);
#pragma unroll
    for (int t = 0; t < 8; ++t) s += v[c].f[t];
  }
  const float mu = cuda::warp_sum(s) * (1.f / h);
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < VPL; ++c)
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float d = v[c].f[t] - mu;
      ss += d * d;
    }
  const float rs = rsqrtf(cuda::warp_sum(ss) * (1.f / h) + 1e-5f);
#pragma unroll
  for (int c = 0; c < VPL; ++c) {
    const int col = (c * 32 + lane) * 8;
    Vec8 gg, bb, o;
    gg.set(graw[c]);
    bb.set(braw[c]);
#pragma unroll
    for (int t = 0; t < 8; ++t) o.f[t] = (v[c].f[t] - mu) * rs * gg.f[t] + bb.f[t];
    o.store(y + (long long)row * h + col);
  }
  if (lane == 0) mean[row] = mu, rstd[row] = rs;
}

template <int VPL>
__global__ void __launch_bounds__(256) k_ln_bwd(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                const float* __restrict__ mean, const float* __restrict__ rstd,
                                                const bf16* __restrict__ g, const bf16* __restrict__ dres,
                                                bf16* __restrict__ dx, float* __restrict__ dgamma,
                                                float* __restrict__ dbeta, float* __restrict__ dsum, int M,
                                                int skip_atomics) {
  cuda::pdl_wait();
  constexpr int h = VPL * 256;
  extern __shared__ float red[];  // [8 warps][2][h] (+ [8 warps][h] column sums of dx when dsum)
  float* colsum = red + 16 * h + (threadIdx.x >> 5) * h;
  if (dsum)
    for (int i = threadIdx.x & 31; i < h; i += 32) colsum[i] = 0.f;  // warp-private slice
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // gamma / beta column partials accumulate in this warp's shared-memory slice (lane-private
  // columns), not registers: 2 x 8 x VPL accumulators per lane had pushed the kernel past
  // 255 registers into local-memory spills
  float* acc = red + warp * 2 * h;  // [gamma | beta][h]
  for (int i = lane * 4; i < 2 * h; i += 128) *reinterpret_cast<float4*>(acc + i) = make_float4(0.f, 0.f, 0.f, 0.f);
  Vec8 gam[VPL];
#pragma unroll
  for (int c = 0; c < VPL; ++c) gam[c].load(g + (c * 32 + lane) * 8);
  // rows are software-pipelined: the next row's dy / x / dres / statistics are in flight
  // (raw 16-byte vectors) while the current one is reduced and written
  const int stride = gridDim.x * 8;
  uint4 nd[VPL], nx[VPL], nr[VPL];
  float nmu = 0.f, nrs = 0.f;
  auto fetch = [&](int r) {
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const long long off = (long long)r * h + (c * 32 + lane) * 8;
      nd[c] = *reinterpret_cast<const uint4*>(dy + off);
      nx[c] = *reinterpret_cast<const uint4*>(x + off);
      nr[c] = dres ? *reinterpret_cast<const uint4*>(dres + off) : make_uint4(0, 0, 0, 0);
    }
    nmu = mean[r];
    nrs = rstd[r];
  };
  int row = blockIdx.x * 8 + warp;
  if (row < M) fetch(row);
  for (; row < M; row += stride) {
    const float mu = nmu, rs = nrs;
    uint4 cd[VPL], cx[VPL], cr[VPL];  // current row, raw (converted per chunk, twice)
#pragma unroll
    for (int c = 0; c < VPL; ++c) cd[c] = nd[c], cx[c] = nx[c], cr[c] = nr[c];
    if (row + stride < M) fetch(row + stride);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      Vec8 dv, xv;
      dv.set(cd[c]);
      xv.set(cx[c]);
      float ag[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float xh = (xv.f[t] - mu) * rs;
        const float gg = dv.f[t] * gam[c].f[t];
        s1 += gg;
        s2 += gg * xh;
        ag[t] = dv.f[t] * xh;
      }
      float4* pg = reinterpret_cast<float4*>(acc + (c * 32 + lane) * 8);
      float4* pb = reinterpret_cast<float4*>(acc + h + (c * 32 + lane) * 8);
      float4 a = pg[0], b = pg[1], u = pb[0], v = pb[1];
      a.x += ag[0], a.y += ag[1], a.z += ag[2], a.w += ag[3];
      b.x += ag[4], b.y += ag[5], b.z += ag[6], b.w += ag[7];
      u.x += dv.f[0], u.y += dv.f[1], u.z += dv.f[2], u.w += dv.f[3];
      v.x += dv.f[4], v.y += dv.f[5], v.z += dv.f[6], v.w += dv.f[7];
      pg[0] = a, pg[1] = b, pb[0] = u, pb[1] = v;
    }
    s1 = cuda::warp_sum(s1) * (1.f / h);
    s2 = cuda::warp_sum(s2) * (1.f / h);
#pragma unroll
    for (int c = 0; c < VPL; ++c) {
      const int col = (c * 32 + lane) * 8;
      Vec8 dv, xv, rv, o;
      dv.set(cd[c]);
      xv.set(cx[c]);
      rv.set(cr[c]);
#pragma unroll
      for (int t = 0; t < 8; ++t)
        o.f[t] = rs * (dv.f[t] * gam[c].f[t] - s1 - (xv.f[t] - mu) * rs * s2) + rv.f[t];
      o.store(dx + (long long)row * h + col);
      if (dsum) {  // column sums of the bf16 dx (the next bias gradient), lane-private smem
        float4* cs = reinterpret_cast<float4*>(colsum + col);
        const Vec8 ob = o.rounded();
        float4 a = cs[0], b = cs[1];
        a.x += ob.f[0], a.y += ob.f[1], a.z += ob.f[2], a.w += ob.f[3];
        b.x += ob.f[4], b.y += ob.f[5], b.z += ob.f[6], b.w += ob.f[7];
        cs[0] = a, cs[1] = b;
      }
    }
  }
  // reduce the per-warp column partials over the 8 warps, then one atomic per column
  __syncthreads();
  // one 16-byte vector atomic per 4 columns (a quarter of the L2 atomic operations)
  auto sum4 = [&](int base, int stride, int col) {
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < 8; ++w) {
      const float4 v = *reinterpret_cast<const float4*>(red + base + w * stride + col);
      a.x += v.x, a.y += v.y, a.z += v.z, a.w += v.w;
    }
    return a;
  };
  if (skip_atomics) return;  // (timing experiment only: CK_LN_BWD_SKIP_ATOMICS)
  for (int col = threadIdx.x * 4; col < h; col += blockDim.x * 4) {
    atomicAdd(reinterpret_cast<float4*>(dgamma + col), sum4(0, 2 * h, col));
    atomicAdd(reinterpret_cast<float4*>(dbeta + col), sum4(h, 2 * h, col));
    if (dsum) atomicAdd(reinterpret_cast<float4*>(dsum + col), sum4(16 * h, h, col));
  }
}

// ------------------------------------------------------------------ embedding --
__global__ void k_embed_fwd(const int32_t* __restrict__ tok, const bf16* __restrict__ wte,
                            const bf16* __restrict__ wpe, bf16* __restrict__ x, int M, int seq, int h) {
  cuda::pdl_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= M) return;
  const bf16* a = wte + (long long)tok[row] * h;
  const bf16* p = wpe + (long long)(row % seq) * h;
  for (int col = lane * 8; col < h; col += 256) {
    Vec8 u, v;
    u.load(a + col);
    v.load(p + col);
#pragma unroll
    for (int t = 0; t < 8; ++t) u.f[t] += v.f[t];
    u.store(x + (long long)row * h + col);
  }
}

__global__ void k_embed_bwd(const int32_t* __restrict__ tok, const bf16* __restrict__ dx,
                            float* __restrict__ dwte, float* __restrict__ dwpe, int M, int seq, int h) {
  cuda::pdl_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= M) return;
  float* a = dwte + (long long)tok[row] * h;
  float* p = dwpe + (long long)(row % seq) * h;
  for (int col = lane * 8; col < h; col += 256) {
    Vec8 u;
    u.load(dx + (long long)row * h + col);
    const float4 lo = make_float4(u.f[0], u.f[1], u.f[2], u.f[3]), hi = make_float4(u.f[4], u.f[5], u.f[6], u.f[7]);
    // 16-byte vector atomics (rows are 16-byte aligned, h % 8 == 0): a quarter of the L2 operations
    atomicAdd(reinterpret_cast<float4*>(a + col), lo), atomicAdd(reinterpret_cast<float4*>(a + col + 4), hi);
    atomicAdd(reinterpret_cast<float4*>(p + col), lo), atomicAdd(reinterpret_cast<float4*>(p + col + 4), hi);
  }
}

// -------------------------------------------------------------- cross-entropy --
// One CTA per row.  Pass 1: online max / sum-exp over the valid V columns (16-byte
// loads); pass 2: in-place gradient.  Vp % 8 == 0.
__global__ void __launch_bounds__(512) k_xent(bf16* __restrict__ logits, long long ld,
                                              const int32_t* __restrict__ labels, int V, int Vp,
                                              float grad_scale, float loss_scale, float* __restrict__ loss_sum) {
  cuda::pdl_wait();
  __shared__ float scratch[32];
  const int row = blockIdx.x;
  bf16* lr = logits + (long long)row * ld;
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x * 8; c < Vp; c += blockDim.x * 8) {
    Vec8 v;
    v.load(lr + c);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (c + t >= V) break;
      const float x = v.f[t];
      if (x > m) s = s * __expf(m - x) + 1.f, m = x;
      else s += __expf(x - m);
    }
  }
  const float gm = cuda::block_max(m, scratch);
  s = (m == -INFINITY) ? 0.f : s * __expf(m - gm);
  const float gs = cuda::block_sum(s, scratch);
  const float lse = gm + __logf(gs);
  const int lab = labels[row];
  const float x_lab = __bfloat162float(lr[lab]);
  __syncthreads();  // everyone has read lr[lab] before it is overwritten
  for (int c = threadIdx.x * 8; c < Vp; c += blockDim.x * 8) {
    Vec8 v;
    v.load(lr + c);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int j = c + t;
      v.f[t] = j < V ? (__expf(v.f[t] - lse) - (j == lab ? 1.f : 0.f)) * grad_scale : 0.f;
    }
    v.store(lr + c);
  }
  if (threadIdx.x == 0) atomicAdd(loss_sum, (lse - x_lab) * loss_scale);
}

// Persistent variant (one 512-thread CTA per SM): rows are streamed into shared memory
// by a 1-D bulk copy one row ahead (double buffer), so the next row's HBM read overlaps
// this row's exps and gradient stores.  Each row is read once and written once (the
// 2 x 2 B per element floor), with one exp per element kept in registers (NV 16-byte
// chunks per thread): max, p = exp(x - max), sum, grad = p / sum - onehot.
template <int NV>
__global__ void __launch_bounds__(512, 1) k_xent_pipe(bf16* __restrict__ logits, long long ld,
                                                      const int32_t* __restrict__ labels, int M, int V, int Vp,
                                                      float grad_scale, float loss_scale, float* __restrict__ loss_sum) {
  extern __shared__ __align__(128) uint8_t xsm[];
  __shared__ float scratch[32];
  __shared__ __align__(8) uint64_t full[2];
  const uint32_t row_bytes = uint32_t(Vp) * 2;
  const uint32_t buf_bytes = (row_bytes + 127) / 128 * 128;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&full[0], 1);
    ptx::mbar_init(&full[1], 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  cuda::pdl_wait();
  cuda::pdl_trigger();
  auto issue = [&](int row, int b) {
    ptx::mbar_arrive_expect_tx(&full[b], row_bytes);
    ptx::bulk_load(xsm + b * buf_bytes, logits + (long long)row * ld, row_bytes, &full[b]);
  };
  if (threadIdx.x == 0 && blockIdx.x < M) issue(blockIdx.x, 0);
  int it = 0;
  for (int row = blockIdx.x; row < M; row += gridDim.x, ++it) {
    const int b = it & 1;
    // the other buffer was last read in the previous iteration (ended by a block barrier)
    if (threadIdx.x == 0 && row + gridDim.x < M) issue(row + gridDim.x, b ^ 1);
    ptx::mbar_wait(&full[b], (it >> 1) & 1);
    const bf16* sr = reinterpret_cast<const bf16*>(xsm + b * buf_bytes);
    bf16* lr = logits + (long long)row * ld;
    const int lab = labels[row];
    float f[NV][8];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 512 + threadIdx.x) * 8;
      Vec8 v;
      if (c < Vp) v.load(sr + c);
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        f[i][t] = (c < Vp && c + t < V) ? v.f[t] : -INFINITY;
        m = fmaxf(m, f[i][t]);
      }
    }
    const float gm = cuda::block_max(m, scratch);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        f[i][t] = __expf(f[i][t] - gm);
        s += f[i][t];
      }
    const float gs = cuda::block_sum(s, scratch);
    const float inv = grad_scale / gs;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 512 + threadIdx.x) * 8;
      if (c >= Vp) continue;
      Vec8 o;
#pragma unroll
      for (int t = 0; t < 8; ++t) o.f[t] = f[i][t] * inv - (c + t == lab ? grad_scale : 0.f);
      o.store(lr + c);
    }
    if (threadIdx.x == 0) atomicAdd(loss_sum, (gm + __logf(gs) - __bfloat162float(sr[lab])) * loss_scale);
    __syncthreads();  // this buffer is free for the row after next
  }
}

// ------------------------------------------------------------------ bias grad --
// CTA = 256 columns x 64 rows: 32 column groups of 8 (16-byte loads) x 8 row lanes;
// per-thread fp32 partials, reduced over the 8 row lanes in shared memory, then one
// atomic per column per CTA.
__global__ void __launch_bounds__(256) k_bias_grad(const bf16* __restrict__ dy, float* __restrict__ db,
                                                   int M, int N) {
  cuda::pdl_wait();
  __shared__ float red[8][256 + 8];
  const int cg = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int col = blockIdx.x * 256 + cg * 8;
  const int r0 = blockIdx.y * 64;
  float acc[8] = {};
  if (col < N) {
    for (int r = r0 + rl; r < min(M, r0 + 64); r += 8) {
      Vec8 v;
      v.load(dy + (long long)r * N + col);
#pragma unroll
      for (int t = 0; t < 8; ++t) acc[t] += v.f[t];
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) red[rl][cg * 8 + t] = acc[t];
  __syncthreads();
  const int c = threadIdx.x;
  if (blockIdx.x * 256 + c < N) {
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += red[k][c];
    atomicAdd(db + blockIdx.x * 256 + c, sum);
  }
}

// -------------------------------------------------------------------- update --
struct GradPtrs {
  float* p[8];
};

template <int COPIES>
__global__ void __launch_bounds__(256) k_sgd(float* __restrict__ w32, bf16* __restrict__ w16, GradPtrs g,
                                             long long n, float lr) {
  cuda::pdl_wait();
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    float4 v[COPIES];
#pragma unroll
    for (int c = 0; c < COPIES; ++c) v[c] = __ldcs(reinterpret_cast<const float4*>(g.p[c] + i));
    float4 w = __ldcs(reinterpret_cast<const float4*>(w32 + i));
    float4 s = v[0];
#pragma unroll
    for (int c = 1; c < COPIES; ++c) s.x += v[c].x, s.y += v[c].y, s.z += v[c].z, s.w += v[c].w;
    w.x -= lr * s.x, w.y -= lr * s.y, w.z -= lr * s.z, w.w -= lr * s.w;
    __stcs(reinterpret_cast<float4*>(w32 + i), w);
    __nv_bfloat162 h[2] = {__floats2bfloat162_rn(w.x, w.y), __floats2bfloat162_rn(w.z, w.w)};
    *reinterpret_cast<uint2*>(w16 + i) = *reinterpret_cast<uint2*>(h);
#pragma unroll
    for (int c = 0; c < COPIES; ++c) __stcs(reinterpret_cast<float4*>(g.p[c] + i), make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

// AdamW (decoupled weight decay, torch.optim.AdamW semantics) over elements [lo, hi) of
// a stage: g = sum of the gradient copies; m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// w = w (1 - lr wd) - lr (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps); w16 = bf16(w);
// the gradients are zeroed.  m / v hold only [lo, hi) (the ZeRO shard: m[i - lo]); the
// step t = *step + 1 is read on the device so one captured graph serves every iteration.
template <int COPIES>
__global__ void __launch_bounds__(256) k_adamw(float* __restrict__ w32, bf16* __restrict__ w16, GradPtrs g,
                                               float* __restrict__ m, float* __restrict__ v, const int* __restrict__ step,
                                               long long lo, long long hi, AdamHP hp) {
  cuda::pdl_wait();
  const float t = float(*step + 1);
  const float c1 = 1.f / (1.f - powf(hp.beta1, t)), c2 = 1.f / (1.f - powf(hp.beta2, t));
  const float decay = 1.f - hp.lr * hp.weight_decay;
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = lo + (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 4; i < hi; i += stride) {
    float4 gs = __ldcs(reinterpret_cast<const float4*>(g.p[0] + i));
#pragma unroll
    for (int c = 1; c < COPIES; ++c) {
      const float4 x = __ldcs(reinterpret_cast<const float4*>(g.p[c] + i));
      gs.x += x.x, gs.y += x.y, gs.z += x.z, gs.w += x.w;
    }
    float4 w = __ldcs(reinterpret_cast<const float4*>(w32 + i));
    float4 mm = __ldcs(reinterpret_cast<const float4*>(m + (i - lo)));
    float4 vv = __ldcs(reinterpret_cast<const float4*>(v + (i - lo)));
    float* wp = &w.x;
    float* mp = &mm.x;
    float* vp = &vv.x;
    const float* gp = &gs.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      mp[e] = hp.beta1 * mp[e] + (1.f - hp.beta1) * gp[e];
      vp[e] = hp.beta2 * vp[e] + (1.f - hp.beta2) * gp[e] * gp[e];
      wp[e] = wp[e] * decay - hp.lr * (mp[e] * c1) / (sqrtf(vp[e] * c2) + hp.eps);
    }
    __stcs(reinterpret_cast<float4*>(w32 + i), w);
    __stcs(reinterpret_cast<float4*>(m + (i - lo)), mm);
    __stcs(reinterpret_cast<float4*>(v + (i - lo)), vv);
    __nv_bfloat162 h[2] = {__floats2bfloat162_rn(w.x, w.y), __floats2bfloat162_rn(w.z, w.w)};
    *reinterpret_cast<uint2*>(w16 + i) = *reinterpret_cast<uint2*>(h);
#pragma unroll
    for (int c = 0; c < COPIES; ++c) __stcs(reinterpret_cast<float4*>(g.p[c] + i), make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

__global__ void k_count_step(int* step) {
  cuda::pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) ++*step;
}

__global__ void k_reduce(float* __restrict__ dst, GradPtrs g, int copies, long long n) {
  cuda::pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < copies; ++c) s += g.p[c][i];
    dst[i] = s;
  }
}

__global__ void k_cast(const float* __restrict__ s, bf16* __restrict__ d, long long n) {
  cuda::pdl_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}

int grid_for(long long n, int per_thread) {
  const long long b = (n / per_thread + 255) / 256;
  return int(b < 148LL * 16 ? (b < 1 ? 1 : b) : 148LL * 16);
}

}  // namespace

void layernorm_fwd(const bf16* x, const bf16* g, const bf16* b, bf16* y, float* mean, float* rstd,
                   int M, int h, cudaStream_t st) {
  const int grid = ceil_div(M, 8);
  switch (h) {
#define CK_LN(V) case V * 256: cuda::launch(k_ln_fwd<V>, dim3(grid), dim3(256), 0, st, x, g, b, y, mean, rstd, M); break;
    CK_LN(1) CK_LN(2) CK_LN(3) CK_LN(4) CK_LN(5) CK_LN(6) CK_LN(8)
#undef CK_LN
    default: throw chimera::capi::InternalError("layernorm: unsupported hidden size");
  }
  CK_CUDA(cudaGetLastError());
}

void layernorm_bwd(const bf16* dy, const bf16* x, const float* mean, const float* rstd, const bf16* g,
                   const bf16* dres, bf16* dx, float* dgamma, float* dbeta, float* dsum, int M, int h,
                   cudaStream_t st) {
  // one 8-warp CTA per SM (255 registers); CK_LN_BWD_RPW=n: at least n rows per warp
  // (fewer CTAs -> fewer column-partial reductions and atomics on small M)
  static const int rpw = [] {
    const char* e = std::getenv("CK_LN_BWD_RPW");
    return e ? std::max(1, atoi(e)) : 1;
  }();
  static const int skip = std::getenv("CK_LN_BWD_SKIP_ATOMICS") ? 1 : 0;
  const int grid = std::min(ceil_div(M, 8 * rpw), cuda::num_sms());
  const size_t smem = size_t(dsum ? 24 : 16) * h * sizeof(float);
  switch (h) {
#define CK_LN(V)                                                                                   \
  case V * 256: {                                                                                  \
    static bool attr = false;                                                                      \
    if (!attr) {                                                                                   \
      CK_CUDA(cudaFuncSetAttribute(k_ln_bwd<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 24 * V * 256 * 4)); \
      attr = true;                                                                                 \
    }                                                                                              \
    cuda::launch(k_ln_bwd<V>, dim3(grid), dim3(256), smem, st, dy, x, mean, rstd, g, dres, dx, dgamma, dbeta, dsum, M, \
                 skip);                                                                            \
    break;                                                                                         \
  }
    CK_LN(1) CK_LN(2) CK_LN(3) CK_LN(4) CK_LN(5) CK_LN(6) CK_LN(8)
#undef CK_LN
    default: throw chimera::capi::InternalError("layernorm: unsupported hidden size");
  }
  CK_CUDA(cudaGetLastError());
}

void embed_fwd(const int32_t* tok, const bf16* wte, const bf16* wpe, bf16* x, int M, int seq, int h,
               cudaStream_t st) {
  cuda::launch(k_embed_fwd, dim3(ceil_div(M, 8)), dim3(256), 0, st, tok, wte, wpe, x, M, seq, h);
  CK_CUDA(cudaGetLastError());
}

void embed_bwd(const int32_t* tok, const bf16* dx, float* dwte, float* dwpe, int M, int seq, int h,
               cudaStream_t st) {
  cuda::launch(k_embed_bwd, dim3(ceil_div(M, 8)), dim3(256), 0, st, tok, dx, dwte, dwpe, M, seq, h);
  CK_CUDA(cudaGetLastError());
}

void xent_fwd_bwd(bf16* logits, long long ld, const int32_t* labels, int M, int V, int Vp,
                  float grad_scale, float loss_scale, float* loss_sum, cudaStream_t st) {
  const int need = ceil_div(Vp, 8 * 512);  // smallest instantiated register footprint that holds the row
  const bool bulk_ok = ld % 8 == 0 && Vp % 8 == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0;
  const int nv = !bulk_ok ? 0 : need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 13 ? 13 : 0;
  const size_t smem = 2 * size_t((Vp * 2 + 127) / 128 * 128);  // two row buffers (<= 208 KB)
  const int grid = std::min(M, cuda::num_sms());
  switch (nv) {
#define CK_XR(NV)                                                                                      \
  case NV: {                                                                                           \
    static bool attr = false;                                                                          \
    if (!attr) {                                                                                       \
      CK_CUDA(cudaFuncSetAttribute(k_xent_pipe<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024)); \
      attr = true;                                                                                     \
    }                                                                                                  \
    cuda::launch(k_xent_pipe<NV>, dim3(grid), dim3(512), smem, st, logits, ld, labels, M, V, Vp, grad_scale, loss_scale, \
                 loss_sum);                                                                            \
    break;                                                                                             \
  }
    CK_XR(1) CK_XR(2) CK_XR(4) CK_XR(8) CK_XR(13)
#undef CK_XR
    default: cuda::launch(k_xent, dim3(M), dim3(512), 0, st, logits, ld, labels, V, Vp, grad_scale, loss_scale, loss_sum);
  }
  CK_CUDA(cudaGetLastError());
}

void bias_grad(const bf16* dy, float* db, int M, int N, cudaStream_t st) {
  if (N % 8) throw chimera::capi::InternalError("bias_grad: N % 8 != 0");
  cuda::launch(k_bias_grad, dim3(ceil_div(N, 256), ceil_div(M, 64)), dim3(256), 0, st, dy, db, M, N);
  CK_CUDA(cudaGetLastError());
}

void sgd_update(float* w32, bf16* w16, float* const* grads, int copies, long long n, float lr,
                cudaStream_t st) {
  if (copies < 1 || copies > 8) throw chimera::capi::InternalError("sgd: 1..8 gradient copies");
  if (n % 4) throw chimera::capi::InternalError("sgd: n % 4 != 0");
  GradPtrs g{};
  for (int c = 0; c < copies; ++c) g.p[c] = grads[c];
  const int grid = grid_for(n, 4);
  switch (copies) {
#define CK_SGD(C) case C: cuda::launch(k_sgd<C>, dim3(grid), dim3(256), 0, st, w32, w16, g, n, lr); break;
    CK_SGD(1) CK_SGD(2) CK_SGD(3) CK_SGD(4) CK_SGD(5) CK_SGD(6) CK_SGD(7) CK_SGD(8)
#undef CK_SGD
  }
  CK_CUDA(cudaGetLastError());
}

void adamw_update(float* w32, bf16* w16, float* const* grads, int copies, float* m, float* v, int* step,
                  long long lo, long long hi, const AdamHP& hp, cudaStream_t st) {
  if (copies < 1 || copies > 8) throw chimera::capi::InternalError("adamw: 1..8 gradient copies");
  if (lo % 4 || hi % 4) throw chimera::capi::InternalError("adamw: range must be a multiple of 4 elements");
  GradPtrs g{};
  for (int c = 0; c < copies; ++c) g.p[c] = grads[c];
  const int grid = grid_for(hi - lo, 4);
  switch (copies) {
#define CK_ADAM(C) \
  case C: cuda::launch(k_adamw<C>, dim3(grid), dim3(256), 0, st, w32, w16, g, m, v, (const int*)step, lo, hi, hp); break;
    CK_ADAM(1) CK_ADAM(2) CK_ADAM(3) CK_ADAM(4) CK_ADAM(5) CK_ADAM(6) CK_ADAM(7) CK_ADAM(8)
#undef CK_ADAM
  }
  cuda::launch(k_count_step, dim3(1), dim3(32), 0, st, step);
  CK_CUDA(cudaGetLastError());
}

void reduce_copies(float* dst, float* const* srcs, int copies, long long n, cudaStream_t st) {
  if (copies < 1 || copies > 8) throw chimera::capi::InternalError("reduce: 1..8 copies");
  GradPtrs g{};
  for (int c = 0; c < copies; ++c) g.p[c] = srcs[c];
  cuda::launch(k_reduce, dim3(grid_for(n, 1)), dim3(256), 0, st, dst, g, copies, n);
  CK_CUDA(cudaGetLastError());
}

void cast_f32_bf16(const float* src, bf16* dst, long long n, cudaStream_t st) {
  cuda::launch(k_cast, dim3(grid_for(n, 1)), dim3(256), 0, st, src, dst, n);
  CK_CUDA(cudaGetLastError());
}

}  // namespace chimera::ops

// ----------------------------------------------------------- C-ABI launchers --
extern "C" {
using chimera::ops::bf16;

CK_API int ck_layernorm_fwd(const void* x, const void* g, const void* b, void* y, float* mean,
                            float* rstd, int M, int h, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::layernorm_fwd((const bf16*)x, (const bf16*)g, (const bf16*)b, (bf16*)y, mean, rstd,
                                M, h, (cudaStream_t)st);
  });
}
CK_API int ck_layernorm_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                            const void* g, const void* dres, void* dx, float* dg, float* db, int M,
                            int h, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::layernorm_bwd((const bf16*)dy, (const bf16*)x, mean, rstd, (const bf16*)g,
                                (const bf16*)dres, (bf16*)dx, dg, db, nullptr, M, h, (cudaStream_t)st);
  });
}
CK_API int ck_layernorm_bwd_dsum(const void* dy, const void* x, const float* mean, const float* rstd,
                                 const void* g, const void* dres, void* dx, float* dg, float* db, float* dsum,
                                 int M, int h, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::layernorm_bwd((const bf16*)dy, (const bf16*)x, mean, rstd, (const bf16*)g,
                                (const bf16*)dres, (bf16*)dx, dg, db, dsum, M, h, (cudaStream_t)st);
  });
}
CK_API int ck_embed_fwd(const int32_t* tok, const void* wte, const void* wpe, void* x, int M, int seq,
                        int h, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::embed_fwd(tok, (const bf16*)wte, (const bf16*)wpe, (bf16*)x, M, seq, h, (cudaStream_t)st);
  });
}
CK_API int ck_embed_bwd(const int32_t* tok, const void* dx, float* dwte, float* dwpe, int M, int seq,
                        int h, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::embed_bwd(tok, (const bf16*)dx, dwte, dwpe, M, seq, h, (cudaStream_t)st);
  });
}
CK_API int ck_xent_fwd_bwd(void* logits, long long ld, const int32_t* labels, int M, int V, int Vp,
                           float grad_scale, float loss_scale, float* loss_sum, void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::xent_fwd_bwd((bf16*)logits, ld, labels, M, V, Vp, grad_scale, loss_scale, loss_sum,
                               (cudaStream_t)st);
  });
}
CK_API int ck_bias_grad(const void* dy, float* db, int M, int N, void* st) {
  return chimera::capi::guarded([&] { chimera::ops::bias_grad((const bf16*)dy, db, M, N, (cudaStream_t)st); });
}
CK_API int ck_sgd_update(float* w32, void* w16, float* const* grads, int copies, long long n, float lr,
                         void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::sgd_update(w32, (bf16*)w16, grads, copies, n, lr, (cudaStream_t)st);
  });
}
}
