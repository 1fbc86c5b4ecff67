// Flash-attention forward on the 5th-generation tensor cores (sm_100a), head dim 64.
//
// CTA = (128-query tile, batch*head); 6 warps:
//   warp 4  TMA producer: Q once, then 128-key K/V tiles into a 2-stage ring
//   warp 5  TMEM allocator + single-thread MMA issuer:
//             S  = Q K^T      tcgen05.mma kind::f16 M128 N128 K64  -> TMEM cols [0,128)
//             O += P V        tcgen05.mma kind::f16 M128 N64  K128 -> TMEM cols [128,192),
//                             A = P straight from TMEM cols [192,256) (bf16 pairs)
//   warps 0-3  softmax: thread t owns query row t (= TMEM lane t): the S row is pulled
//             into registers in one pass, which frees the S columns at once (s_free) so
//             the MMA warp computes S_{j+1} underneath this tile's exp2s; P goes back to
//             TMEM as bf16 pairs (tcgen05.st) for the PV MMA, running O is rescaled in
//             TMEM only when a row max moves by more than 2^8; final O / l is staged
//             in the item's consumed Q buffer and leaves by one TMA store (row tails:
//             per-thread stores), the log-sum-exp per thread.
// Persistent: (query tile, batch*head) items, heaviest first, dealt boustrophedon-wise.
// The Q/K/V tiles come straight out of the packed [tokens, 3*H*64] QKV GEMM output via
// one 2-D TMA map (no head split), so the kernel reads exactly Q, K, V once per tile.
// ~96 KB smem and 256 TMEM columns per CTA: two CTAs per SM overlap one CTA's softmax
// with the other's MMAs.
#include <cuda.h>

#include "chimera_ck.h"
#include "common.cuh"
#include "ops.cuh"
#include "ptx_sm100.cuh"
#include "tma_host.hpp"

namespace chimera::ops {

// Per-phase clock64() stamps of CTA 0 (scripts/attn_trace.cu builds with CK_ATTN_TRACE).
#ifdef CK_ATTN_TRACE
__device__ long long g_attn_trace[32][16];
__device__ int g_attn_trace_cta = 0;  // the CTA whose phases are stamped
__device__ long long g_attn_warp[2][32][16];  // per-warp stamps [kind][tile][warp]
#define ATTN_WTRACE(kind, j)                                                                       \
  do {                                                                                              \
    if ((threadIdx.x & 31) == 0 && blockIdx.x == g_attn_trace_cta && (j) < 32)                     \
      g_attn_warp[kind][j][threadIdx.x >> 5] = clock64();                                          \
  } while (0)
__device__ long long g_attn_cta[4096][3];  // smid, globaltimer at entry / exit
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ int smid() {
  int v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
#define ATTN_CTA(slot) \
  if (threadIdx.x == 0 && blockIdx.x < 4096) g_attn_cta[blockIdx.x][slot] = slot == 0 ? smid() : gtimer()
#define ATTN_TRACE(cond, j, ev)                                                  \
  do {                                                                           \
    if ((cond) && blockIdx.x == g_attn_trace_cta && (j) < 32) g_attn_trace[j][ev] = clock64(); \
  } while (0)
#else
#define ATTN_TRACE(cond, j, ev) \
  do {                          \
  } while (0)
#define ATTN_WTRACE(kind, j) \
  do {                       \
  } while (0)
#define ATTN_CTA(slot)
#endif

namespace {

using ptx::ex2_approx;
constexpr int kQ = 128, kKV = 128, kD = 64;
constexpr int kTileBytes = kQ * kD * 2;  // 16 KB: 128 rows x 128 B
constexpr int kSmemQ = 0, kSmemK = 2 * kTileBytes, kSmemV = 4 * kTileBytes;  // Q[2], K[2], V[2]
constexpr int kSmemBar = 6 * kTileBytes;
constexpr int kSmemTotal = kSmemBar + 256;
constexpr float kLog2e = 1.4426950408889634f;
// Share of the softmax exp2s computed by ptx::ex2_poly2 on the FMA pipes: every
// kPolyEvery-th pair (0 = all on MUFU).  The forward is MUFU-bound at head dim 64
// (16 ex2/clk/SM vs 128x128 exps per tile): one pair in three off MUFU measured -6%.
#ifndef CK_ATTN_POLY_EVERY
#define CK_ATTN_POLY_EVERY 3
#endif
constexpr int kPolyEvery = CK_ATTN_POLY_EVERY;

// The MMA issuer sits on the critical path of every hand-off (P ready -> PV, dS ready
// -> dV/dK/dQ): it polls (try_wait) instead of sleeping, whose wake-up costs ~400 cycles.
#ifndef CK_ATTN_MMA_SPIN
#define CK_ATTN_MMA_SPIN 1
#endif
__device__ __forceinline__ void mma_wait(uint64_t* bar, uint32_t parity) {
  if (CK_ATTN_MMA_SPIN) ptx::mbar_wait(bar, parity);
  else ptx::mbar_wait_sleep(bar, parity);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// The CTA's sequence of (query tile item, key tile) iterations: items (qb, batch*head)
// heaviest first (under causal masking the last query tiles see the most key tiles),
// dealt boustrophedon-wise over the persistent CTAs.
struct FwdSeq {
  int G, c, n_items, BH, nq;
  bool causal;
  int r = 0, n = 0;  // round, item ordinal within this CTA
  int item = -1, qb = 0, bh = 0, nkb = 0, j = 0;
  __device__ int item_of(int rr) const {
    const int i = rr * G + ((rr & 1) ? G - 1 - c : c);
    return i < n_items ? i : -1;
  }
  __device__ void load() {
    item = item_of(r);
    if (item < 0) return;
    const int tile = item / BH;
    bh = item % BH, qb = causal ? nq - 1 - tile : tile, nkb = causal ? qb + 1 : nq, j = 0;
  }
  __device__ bool valid() const { return item >= 0; }
  __device__ void advance() {
    if (++j == nkb) {
      ++r, ++n;
      load();
    }
  }
};

// Persistent: two CTAs per SM, each walking its items; the next item's Q lands in the
// second Q buffer and its first S MMA runs while the current item's O is written out.
template <bool CAUSAL>
__global__ void __launch_bounds__(192, 2)
    k_attn_fwd_tc(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tout,
                  bf16* __restrict__ out, float* __restrict__ lse, int seq, int H, int BH) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((ptx::smem_u32(smem) & 1023) != 0) __trap();  // swizzle atoms need 1 KB alignment
  ATTN_CTA(0);
  ATTN_CTA(1);
  ATTN_TRACE(threadIdx.x == 0, 0, 14);  // entry
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kSmemBar);
  // K and V have separate full / empty barriers: K_j's slot frees when S_j's MMA is done
  // (not after P_j V_j), so the producer loads K two tiles ahead and the S MMA never waits
  // on the TMA (measured: with one K+V barrier pair ~570 of the ~2500 cycles per tile went
  // to waiting for K, scripts/attn_trace.cu)
  uint64_t *q_full = bar, *q_empty = bar + 2, *k_full = bar + 4, *k_empty = bar + 6, *s_full = bar + 8,
           *p_full = bar + 9, *o_done = bar + 10, *s_free = bar + 11, *o_free = bar + 12, *v_full = bar + 13,
           *v_empty = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = (seq + kQ - 1) / kQ;
  FwdSeq seq0;
  seq0.G = gridDim.x, seq0.c = blockIdx.x, seq0.n_items = nq * BH, seq0.BH = BH, seq0.nq = nq, seq0.causal = CAUSAL;
  seq0.load();

  if (warp == 4 && lane == 0) {
    ptx::tma_prefetch(&tqkv);
    ptx::tma_prefetch(&tout);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&q_full[s], 1), ptx::mbar_init(&q_empty[s], 1);
      ptx::mbar_init(&k_full[s], 1), ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1), ptx::mbar_init(&v_empty[s], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(p_full, 128);
    ptx::mbar_init(o_done, 1);
    ptx::mbar_init(s_free, 128);
    ptx::mbar_init(o_free, 128);
    ptx::fence_barrier_init();
  }
  if (warp == 5) ptx::tmem_alloc(tmem_slot, 256);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S: cols [0,128), O: [128,192), P (bf16 pairs): [192,256)
  ATTN_TRACE(threadIdx.x == 0, 1, 14);  // set-up done
  cuda::pdl_wait();
  cuda::pdl_trigger();
  ATTN_TRACE(threadIdx.x == 0, 2, 14);  // dependency resolved

  if (warp == 4) {
    if (lane == 0) {
      int g = 0;
      for (FwdSeq q = seq0; q.valid();) {
        const int b = q.bh / H, hd = q.bh % H, row_base = b * seq, qbuf = q.n & 1;
        ptx::mbar_wait_sleep(&q_empty[qbuf], ((q.n >> 1) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&q_full[qbuf], kTileBytes);
        ptx::tma_load_2d(smem + kSmemQ + qbuf * kTileBytes, &tqkv, &q_full[qbuf], hd * kD, row_base + q.qb * kQ);
        const int n0 = q.n;
        while (q.valid() && q.n == n0) {
          const int st = g & 1;
          ptx::mbar_wait_sleep(&k_empty[st], ((g >> 1) & 1) ^ 1);
          ATTN_TRACE(true, g, 0);
          ptx::mbar_arrive_expect_tx(&k_full[st], kTileBytes);
          ptx::tma_load_2d(smem + kSmemK + st * kTileBytes, &tqkv, &k_full[st], H * kD + hd * kD,
                           row_base + q.j * kKV);
          ptx::mbar_wait_sleep(&v_empty[st], ((g >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&v_full[st], kTileBytes);
          ptx::tma_load_2d(smem + kSmemV + st * kTileBytes, &tqkv, &v_full[st], 2 * H * kD + hd * kD,
                           row_base + q.j * kKV);
          ++g;
          q.advance();
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0 && seq0.valid()) {
      constexpr uint32_t id_s = ptx::idesc_bf16(kQ, kKV, false, false);
      constexpr uint32_t id_o = ptx::idesc_bf16(kQ, kD, false, true);
      auto issue_s = [&](int g, int n, bool first_of_item) {
        const int st = g & 1, qbuf = n & 1;
        if (first_of_item) mma_wait(&q_full[qbuf], (n >> 1) & 1);
        mma_wait(&k_full[st], (g >> 1) & 1);
        ATTN_TRACE(true, g, 1);
        ptx::tc_fence_after();
        const uint32_t sq = ptx::smem_u32(smem + kSmemQ + qbuf * kTileBytes);
        const uint32_t sk = ptx::smem_u32(smem + kSmemK + st * kTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k)
          ptx::umma_f16(tmem, ptx::smem_desc_sw128(sq + k * 32, 16, 1024), ptx::smem_desc_sw128(sk + k * 32, 16, 1024),
                        id_s, k > 0);
        ptx::umma_commit(s_full);
        ptx::umma_commit(&k_empty[st]);  // K_g is read once: free its slot with S_g
      };
      issue_s(0, 0, true);
      int g = 0;
      for (FwdSeq q = seq0; q.valid(); ++g) {
        const int n = q.n, j = q.j;
        FwdSeq nx = q;
        nx.advance();
        // S_g is in the softmax registers: compute the next scores now -- except at an item
        // boundary, where the item's last P V goes first (its O epilogue is the softmax
        // warps' next step; the next item's S may still wait for that item's Q)
        const bool s_first = nx.valid() && nx.n == n;
        if (s_first) {
          mma_wait(s_free, g & 1);
          ATTN_TRACE(true, g, 2);
          ptx::tc_fence_after();
          issue_s(g + 1, nx.n, false);
        }
        mma_wait(p_full, g & 1);  // P_g in TMEM, O rescaled
        ATTN_TRACE(true, g, 3);
        if (j == 0 && n > 0) mma_wait(o_free, (n - 1) & 1);  // previous item's O read out
        mma_wait(&v_full[g & 1], (g >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t sv = ptx::smem_u32(smem + kSmemV + (g & 1) * kTileBytes);
#pragma unroll
        for (int k = 0; k < kKV / 16; ++k)  // A = P from TMEM cols [192, 256): 16 keys = 8 columns
          ptx::umma_f16_ts(tmem + 128, tmem + 192 + k * 8, ptx::smem_desc_sw128(sv + k * 2048, kTileBytes, 1024), id_o,
                           (j > 0 || k > 0) ? 1u : 0u);
        ptx::umma_commit(&v_empty[g & 1]);
        ptx::umma_commit(o_done);
        ATTN_TRACE(true, g, 13);  // PV_g issued
        if (nx.valid() && !s_first) {
          mma_wait(s_free, g & 1);
          ATTN_TRACE(true, g, 2);
          ptx::tc_fence_after();
          issue_s(g + 1, nx.n, true);
        }
        q = nx;
      }
    }
  } else {
    // softmax warps: thread t owns query row t (= TMEM lane t)
    const int t = threadIdx.x;  // 0..127
    const uint32_t trow = tmem + (uint32_t(warp * 32) << 16);
    const float sl2 = 0.125f * kLog2e;
    float m = -INFINITY, l = 0.f;
    // O of a whole query tile leaves through a TMA store staged in the item's (consumed) Q
    // buffer; thread 0 frees that buffer (q_empty) once the store has read it, one tile
    // later, so the warps never wait for the store
    int pend_buf = -1;
    int g = 0;
    for (FwdSeq q = seq0; q.valid(); ++g) {
      const int b = q.bh / H, hd = q.bh % H, row_base = b * seq;
      const int q0 = q.qb * kQ, qr = q0 + t, j = q.j;
      const bool last = j + 1 == q.nkb;
      if (j == 0) m = -INFINITY, l = 0.f;
      ATTN_TRACE(t == 0, g, 4);
      ptx::mbar_wait(s_full, g & 1);
      ATTN_TRACE(t == 0, g, 5);
      ptx::tc_fence_after();
      const int key0 = j * kKV;
      // the whole 128-score row lives in registers (one TMEM pass)
      uint32_t r[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) ptx::tmem_ld32(trow + c * 32, r[c]);
      ptx::tmem_ld_wait();
      ATTN_TRACE(t == 0, g, 6);
      ATTN_TRACE(t == 32, g, 10);  // the other softmax warps' S loads (s_free needs all 128)
      ATTN_TRACE(t == 64, g, 11);
      ATTN_TRACE(t == 96, g, 12);
      ptx::tc_fence_before();
      ptx::mbar_arrive(s_free);
      // masking only on the diagonal (causal) / sequence-tail tile (warp-uniform branch):
      // keys past `lim` (tile-relative) drop out as raw -inf scores
      if ((CAUSAL && key0 + kKV - 1 > q0) || key0 + kKV > seq) {
        const int lim = CAUSAL ? min(qr - key0, seq - 1 - key0) : seq - 1 - key0;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (c * 32 + i > lim) r[c][i] = 0xff800000u;
      }
      // row max on the raw scores (the 1/sqrt(d)*log2(e) scale is applied inside the
      // exp2 FMA below); 8 independent chains
      // three-input max (FMNMX3 on sm_100a): 64 instructions for the 128 scores
      float mxp[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mxp[u] = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; i += 2)
          asm("max.f32 %0, %1, %2, %3;"
              : "=f"(mxp[(i >> 1) & 7])
              : "f"(mxp[(i >> 1) & 7]), "f"(__uint_as_float(r[c][i])), "f"(__uint_as_float(r[c][i + 1])));
      const float mx = fmaxf(fmaxf(fmaxf(mxp[0], mxp[1]), fmaxf(mxp[2], mxp[3])),
                             fmaxf(fmaxf(mxp[4], mxp[5]), fmaxf(mxp[6], mxp[7]))) * sl2;
      // the running max only moves when the new one exceeds it by more than 2^8 (P <= 256
      // is exact enough in fp32 / bf16), so the O rescale below almost never runs
      const float mn = mx > m + 8.f ? mx : m;
      const float safe = mn == -INFINITY ? 0.f : mn;
      const float alpha = ex2_approx(m - safe);
      m = mn;
      l *= alpha;
      ATTN_TRACE(t == 0, g, 7);
      // P = exp2(s * scale - m) -> bf16 pairs in registers first, so that the previous
      // P V (which still reads the P columns and writes O) completes underneath
      const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-safe, -safe);
      float2 ls[4] = {};  // independent packed sum chains
      uint32_t pk[64];
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 x = ptx::fma2(make_float2(__uint_as_float(r[c][i]), __uint_as_float(r[c][i + 1])), sc2, nm2);
          // every kPolyEvery-th pair on the FMA pipes, the rest on MUFU
          const float2 p = (kPolyEvery > 0 && (i >> 1) % (kPolyEvery > 0 ? kPolyEvery : 1) == kPolyEvery - 1)
                               ? ptx::ex2_poly2(x)
                               : make_float2(ex2_approx(x.x), ex2_approx(x.y));
          ls[(i >> 1) & 3] = ptx::add2(ls[(i >> 1) & 3], p);
          __nv_bfloat162 hb = __floats2bfloat162_rn(p.x, p.y);
          pk[c * 16 + (i >> 1)] = *reinterpret_cast<uint32_t*>(&hb);
        }
      {
        const float2 s01 = ptx::add2(ptx::add2(ls[0], ls[1]), ptx::add2(ls[2], ls[3]));
        l += s01.x + s01.y;
      }
      if (g > 0) {  // the previous P V must have read P (and, within the item, written O)
        ptx::mbar_wait(o_done, (g - 1) & 1);
        ATTN_TRACE(t == 0, g, 8);
        ptx::tc_fence_after();
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {  // rescale only when a row max moved
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            ptx::tmem_ld32(trow + 128 + c * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float2 v = ptx::mul2(make_float2(__uint_as_float(o[i]), __uint_as_float(o[i + 1])),
                                         make_float2(alpha, alpha));
              o[i] = __float_as_uint(v.x);
              o[i + 1] = __float_as_uint(v.y);
            }
            tmem_st32(trow + 128 + c * 32, o);
          }
          tmem_st_wait();
        }
      }
      // P (bf16 pairs) into TMEM cols [192, 256) of this row: the PV MMA's A operand
      tmem_st32(trow + 192, *reinterpret_cast<const uint32_t(*)[32]>(pk));
      tmem_st32(trow + 224, *reinterpret_cast<const uint32_t(*)[32]>(pk + 32));
      tmem_st_wait();
      ATTN_TRACE(t == 0, g, 9);
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full);
      if (t == 0 && pend_buf >= 0) {
        ptx::bulk_wait_read0();
        ptx::mbar_arrive(&q_empty[pend_buf]);
        pend_buf = -1;
      }
      if (last) {  // item epilogue: O / l -> bf16, log-sum-exp
        ptx::mbar_wait(o_done, g & 1);
        ptx::tc_fence_after();
        uint32_t o[2][32];
        ptx::tmem_ld32(trow + 128, o[0]);
        ptx::tmem_ld32(trow + 160, o[1]);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(o_free);
        const float inv = l > 0.f ? 1.f / l : 0.f;
        const int qbuf = q.n & 1;
        if (q0 + kQ <= seq) {  // whole tile: swizzled stage in the Q buffer -> TMA store
          uint8_t* stg = smem + kSmemQ + qbuf * kTileBytes;
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            uint32_t pk4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int jj = g8 * 8 + 2 * e;
              __nv_bfloat162 hb = __floats2bfloat162_rn(__uint_as_float(o[jj >> 5][jj & 31]) * inv,
                                                        __uint_as_float(o[jj >> 5][(jj & 31) + 1]) * inv);
              pk4[e] = *reinterpret_cast<uint32_t*>(&hb);
            }
            *reinterpret_cast<uint4*>(stg + t * 128 + ((g8 ^ (t & 7)) << 4)) = make_uint4(pk4[0], pk4[1], pk4[2], pk4[3]);
          }
          ptx::fence_proxy_async();
          asm volatile("bar.sync 1, 128;" ::: "memory");
          if (t == 0) {
            ptx::tma_store_2d(&tout, stg, hd * kD, row_base + q0);
            ptx::bulk_commit();
            pend_buf = qbuf;
          }
          lse[(long long)q.bh * seq + qr] = (m + __log2f(l)) / kLog2e;
        } else {
          if (t == 0) ptx::mbar_arrive(&q_empty[qbuf]);  // the S MMAs are done with this Q
        }
        if (q0 + kQ > seq && qr < seq) {
          bf16* orow = out + ((long long)row_base + qr) * (H * kD) + hd * kD;
#pragma unroll
          for (int g8 = 0; g8 < 8; ++g8) {
            uint32_t pk4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int jj = g8 * 8 + 2 * e;
              __nv_bfloat162 hb = __floats2bfloat162_rn(__uint_as_float(o[jj >> 5][jj & 31]) * inv,
                                                        __uint_as_float(o[jj >> 5][(jj & 31) + 1]) * inv);
              pk4[e] = *reinterpret_cast<uint32_t*>(&hb);
            }
            *reinterpret_cast<uint4*>(orow + g8 * 8) = make_uint4(pk4[0], pk4[1], pk4[2], pk4[3]);
          }
          lse[(long long)q.bh * seq + qr] = (m + __log2f(l)) / kLog2e;
        }
      }
      q.advance();
    }
    if (t == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
  ATTN_CTA(2);
}

// ----------------------------------------------------------------- backward --
// Persistent: one CTA per SM walks its share of the (128-key tile, batch*head) work
// items -- heaviest first (key tile 0 sees every query tile under causal masking),
// dealt boustrophedon-wise over the CTAs (the order balances like dynamic LPT) --
// and pipelines across items: the next item's K/V land in the second K/V buffer and
// its first S/dP MMAs run while the current item's dK/dV are written out.  16 warps:
//   warp 8   TMA producer: per item K, V (2 buffers); per 128-query tile Q and dO
//            (2-stage ring)
//   warp 9   TMEM allocator + single-thread MMA issuer
//   warps 0-7  two compute warpgroups; warp w reads TMEM lanes 32*(w%4).. (thread <->
//            query row), WG g owns key columns [64g, 64g+64) of every tile, so the
//            row's log-sum-exp and D are two per-thread scalars
// Per query tile (global iteration counter g runs across items):
//   S  = Q K^T, dP = dO V^T          (M128 q, N128 keys, K64)  TMEM [0,128), [128,256);
//     issued as soon as the previous tile's S / dP sit in registers (st_free)
//   P = exp2(S c - lse2), dS = P (dP - D) -> bf16, 128-byte-swizzled [q][key] smem tiles
//     (each WG writes its own 64-key block); dS also -> TMEM [448,512) as bf16 pairs
//   dV += P^T dO, dK += dS^T Q       (M128 keys, N64, K128 q)  TMEM [256,320), [320,384)
//     -- P / dS read from smem as MN-major A operands
//   dQ_g = dS K                      (M128 q, N64, K128 keys)  TMEM [384,448), A = dS
//     from TMEM (kDsTmem; CK_ATTN_DS_TMEM=0: dS from smem, dQ double-buffered in
//     [384 + 64 (g&1), ..)).  The tile's lse / D rows arrive with Q / dO (bulk copies).
//   dQ_g is drained by a 4th warpgroup (warps 12-15, one per TMEM lane quarter) as soon
//   as its MMA completes (dq_full), underneath the compute warpgroups' next tile:
//   TMEM -> swizzled smem stage -> two TMA bulk tensor reduce-adds into the fp32 dQ
//   accumulator (no per-thread atomics).  Draining it in the compute warps cost ~1.3 k
//   of the ~3.6 k cycles per tile on their critical path.  setmaxnreg moves registers
//   from the TMA/MMA and drain warpgroups (64) to the compute ones (192).
// Item epilogue: dK (x 1/sqrt(d)) / dV leave TMEM (acc_free lets the next item's MMAs
// accumulate), are staged bf16 in the WG's P tile (free once the item's last MMAs are
// done) and written by TMA stores.
constexpr int kB_K = 0, kB_V = 2 * kTileBytes, kB_Q = 4 * kTileBytes, kB_DO = 6 * kTileBytes,
              kB_P = 8 * kTileBytes, kB_DS = 10 * kTileBytes, kB_DQ = 12 * kTileBytes;  // stage [WG][128][128 B]
constexpr int kB_BAR = 14 * kTileBytes;
// per query-tile stage: the tile's 128 log-sum-exp and D values, bulk-copied with Q / dO
// (on the same full barrier) so the compute warps read them from shared memory -- a
// global load hoisted by the scheduler had stalled them ~1/5 of the time (ncu r02ai)
constexpr int kB_LSE = kB_BAR + 256;  // [2 stages][lse, D][128] fp32
constexpr int kBwdSmem = kB_LSE + 2 * 2 * kQ * 4;
constexpr int kBwdThreads = 512;  // WG0-1 compute, WG2 = TMA + MMA warps, WG3 dQ drain
// Register split per SM sub-partition (one warp of each warpgroup): 2 x 192 + 64 + 64 = 512.
constexpr int kBwdRegsCompute = 192, kBwdRegsOther = 64;
#ifndef CK_ATTN_BWD_POLY_EVERY  // backward: not MUFU-bound, the polynomial costs more than it saves
#define CK_ATTN_BWD_POLY_EVERY 0
#endif
constexpr int kBwdPolyEvery = CK_ATTN_BWD_POLY_EVERY;
#ifndef CK_ATTN_DQ_RED  // 1: dQ drained by vector reductions from registers; 0: smem stage + TMA reduce-add
#define CK_ATTN_DQ_RED 0
#endif
constexpr bool kDqRed = CK_ATTN_DQ_RED != 0;
// 1: the dQ MMA takes dS from TMEM (compute warps tcgen05.st it beside the smem copy the
// dK MMA reads transposed), the dQ accumulator single-buffered to make room: 32 KB less
// shared-memory operand traffic per tile, the resource this kernel is bound by
#ifndef CK_ATTN_DS_TMEM
#define CK_ATTN_DS_TMEM 1
#endif
constexpr bool kDsTmem = CK_ATTN_DS_TMEM != 0;
// dQ accumulator buffer / barrier slot of tile g and the parity of its full phase
__device__ __forceinline__ int dq_slot(int g) { return kDsTmem ? 0 : (g & 1); }
__device__ __forceinline__ uint32_t dq_full_parity(int g) { return kDsTmem ? (g & 1) : ((g >> 1) & 1); }

__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// The CTA's sequence of (item, query tile) iterations.
struct BwdSeq {
  int G, c, n_items, BH, nk, nq;
  bool causal;
  int r = 0, n = 0;          // round, item ordinal within this CTA
  int item = -1, kb = 0, bh = 0, j0 = 0, niter = 0, it = 0;
  __device__ int item_of(int rr) const {
    const int i = rr * G + ((rr & 1) ? G - 1 - c : c);
    return i < n_items ? i : -1;
  }
  __device__ void load() {
    item = item_of(r);
    if (item < 0) return;
    kb = item / BH, bh = item % BH, j0 = causal ? kb : 0, niter = nq - j0, it = 0;
  }
  __device__ bool valid() const { return item >= 0; }
  __device__ void advance() {  // next query tile (possibly of the next item)
    if (++it == niter) {
      ++r, ++n;
      load();
    }
  }
};

template <bool CAUSAL>
__global__ void __launch_bounds__(kBwdThreads, 1)
    k_attn_bwd_tc(const __grid_constant__ CUtensorMap tqkv, const __grid_constant__ CUtensorMap tdo,
                  const __grid_constant__ CUtensorMap tdq, const __grid_constant__ CUtensorMap tdqkv,
                  const float* __restrict__ lse, const float* __restrict__ Dv, bf16* __restrict__ dqkv, int seq, int H,
                  int BH, float* __restrict__ dbias, int lse_bulk, float* __restrict__ dqacc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((ptx::smem_u32(smem) & 1023) != 0) __trap();
  ATTN_CTA(0);
  ATTN_CTA(1);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kB_BAR);
  uint64_t *kv_full = bar, *kv_empty = bar + 2, *qd_full = bar + 4, *qd_empty = bar + 6, *s_full = bar + 8,
           *st_free = bar + 9, *ds_full = bar + 10, *mm_done = bar + 11, *dq_free = bar + 12,  // [2]
      *acc_free = bar + 14, *dq_full = bar + 16;  // dq_full [2]: dQ_g in TMEM buffer g & 1
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 15);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (seq + kKV - 1) / kKV, nq = (seq + kQ - 1) / kQ;
  BwdSeq seq0;
  seq0.G = gridDim.x, seq0.c = blockIdx.x, seq0.n_items = nk * BH, seq0.BH = BH, seq0.nk = nk, seq0.nq = nq;
  seq0.causal = CAUSAL;
  seq0.load();

  if (warp == 8 && lane == 0) {
    ptx::tma_prefetch(&tqkv);
    ptx::tma_prefetch(&tdo);
    ptx::tma_prefetch(&tdq);
    ptx::tma_prefetch(&tdqkv);
    for (int b2 = 0; b2 < 2; ++b2) {
      ptx::mbar_init(&kv_full[b2], 1), ptx::mbar_init(&kv_empty[b2], 1);
      ptx::mbar_init(&qd_full[b2], 1), ptx::mbar_init(&qd_empty[b2], 1);
      ptx::mbar_init(&dq_free[b2], 128);
      ptx::mbar_init(&dq_full[b2], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(st_free, 256);
    ptx::mbar_init(ds_full, 256);
    ptx::mbar_init(mm_done, 1);
    ptx::mbar_init(acc_free, 256);
    ptx::fence_barrier_init();
  }
  if (warp == 9) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cuda::pdl_wait();
  cuda::pdl_trigger();
  constexpr uint32_t kS = 0, kDP = 128, kDV = 256, kDK = 320, kDQ = 384, kDS = 448;  // kDS: dS bf16 pairs (kDsTmem)

  // setmaxnreg is warpgroup-aligned: one instruction for warps 8-15 (TMA, MMA, two idle,
  // the drain warpgroup), one for the compute warpgroups, each heading its role block
  if (warp >= 8) {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kBwdRegsOther));
  if (warp == 8) {
    if (lane == 0) {
      int g = 0;
      for (BwdSeq q = seq0; q.valid();) {
        const int b = q.bh / H, hd = q.bh % H, row_base = b * seq;
        const int kvb = q.n & 1, u = q.n >> 1;
        ptx::mbar_wait_sleep(&kv_empty[kvb], (u & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(&kv_full[kvb], 2 * kTileBytes);
        ptx::tma_load_2d(smem + kB_K + kvb * kTileBytes, &tqkv, &kv_full[kvb], H * kD + hd * kD, row_base + q.kb * kKV);
        ptx::tma_load_2d(smem + kB_V + kvb * kTileBytes, &tqkv, &kv_full[kvb], 2 * H * kD + hd * kD,
                         row_base + q.kb * kKV);
        const int n0 = q.n;
        while (q.valid() && q.n == n0) {
          const int st = g & 1, q0 = (q.j0 + q.it) * kQ;
          // lse / D rows of the tile (seq % 4 == 0: 16-byte aligned, whole 16-byte rows)
          const uint32_t lb = lse_bulk ? uint32_t(min(kQ, seq - q0)) * 4u : 0u;
          ptx::mbar_wait_sleep(&qd_empty[st], ((g >> 1) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&qd_full[st], 2 * kTileBytes + 2 * lb);
          ptx::tma_load_2d(smem + kB_Q + st * kTileBytes, &tqkv, &qd_full[st], hd * kD, row_base + q0);
          ptx::tma_load_2d(smem + kB_DO + st * kTileBytes, &tdo, &qd_full[st], hd * kD, row_base + q0);
          if (lb) {
            const long long o = (long long)q.bh * seq + q0;
            ptx::bulk_load(smem + kB_LSE + st * 1024, lse + o, lb, &qd_full[st]);
            ptx::bulk_load(smem + kB_LSE + st * 1024 + 512, Dv + o, lb, &qd_full[st]);
          }
          ++g;
          q.advance();
        }
      }
    }
  } else if (warp == 9) {
    if (lane == 0 && seq0.valid()) {
      constexpr uint32_t id_s = ptx::idesc_bf16(128, 128, false, false);
      constexpr uint32_t id_kv = ptx::idesc_bf16(128, 64, true, true);  // A = P^T / dS^T (MN-major), B MN-major
      constexpr uint32_t id_q = ptx::idesc_bf16(128, 64, false, true);  // A = dS (K-major), B = K (MN-major)
      const uint32_t sp = ptx::smem_u32(smem + kB_P), sds = ptx::smem_u32(smem + kB_DS);
      // S / dP of iteration (g, item ordinal n) -- waits for that item's K/V the first time
      auto issue_s = [&](int g, int n, bool first_of_item) {
        const int st = g & 1, kvb = n & 1;
        if (first_of_item) mma_wait(&kv_full[kvb], (n >> 1) & 1);
        mma_wait(&qd_full[st], (g >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t sk = ptx::smem_u32(smem + kB_K + kvb * kTileBytes);
        const uint32_t sv = ptx::smem_u32(smem + kB_V + kvb * kTileBytes);
        const uint32_t sq = ptx::smem_u32(smem + kB_Q + st * kTileBytes);
        const uint32_t sdo = ptx::smem_u32(smem + kB_DO + st * kTileBytes);
#pragma unroll
        for (int k = 0; k < kD / 16; ++k) {
          ptx::umma_f16(tmem + kS, ptx::smem_desc_sw128(sq + k * 32, 16, 1024), ptx::smem_desc_sw128(sk + k * 32, 16, 1024),
                        id_s, k > 0);
          ptx::umma_f16(tmem + kDP, ptx::smem_desc_sw128(sdo + k * 32, 16, 1024),
                        ptx::smem_desc_sw128(sv + k * 32, 16, 1024), id_s, k > 0);
        }
        ptx::umma_commit(s_full);
      };
      issue_s(0, 0, true);
      int g = 0;
      for (BwdSeq q = seq0; q.valid(); ++g) {
        const int st = g & 1, n = q.n, kvb = n & 1, it = q.it;
        const bool last = it + 1 == q.niter;
        BwdSeq nx = q;
        nx.advance();
        if (nx.valid()) {  // this tile's S / dP are in registers: next tile's scores now
          mma_wait(st_free, g & 1);
          ptx::tc_fence_after();
          issue_s(g + 1, nx.n, nx.n != n);
          ATTN_TRACE(true, g, 4);
        }
        const uint32_t sk = ptx::smem_u32(smem + kB_K + kvb * kTileBytes);
        const uint32_t sq = ptx::smem_u32(smem + kB_Q + st * kTileBytes);
        const uint32_t sdo = ptx::smem_u32(smem + kB_DO + st * kTileBytes);
        mma_wait(ds_full, g & 1);  // P, dS of this tile in smem
        ATTN_TRACE(true, g, 1);
        if (it == 0 && n > 0) mma_wait(acc_free, (n - 1) & 1);  // previous item's dK / dV read out
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kQ / 16; ++k) {  // reduce over 16 queries per step
          const uint64_t a_p = ptx::smem_desc_sw128(sp + k * 2048, kTileBytes, 1024);
          const uint64_t a_ds = ptx::smem_desc_sw128(sds + k * 2048, kTileBytes, 1024);
          ptx::umma_f16(tmem + kDV, a_p, ptx::smem_desc_sw128(sdo + k * 2048, kTileBytes, 1024), id_kv,
                        (it > 0 || k > 0) ? 1u : 0u);
          ptx::umma_f16(tmem + kDK, a_ds, ptx::smem_desc_sw128(sq + k * 2048, kTileBytes, 1024), id_kv,
                        (it > 0 || k > 0) ? 1u : 0u);
        }
        ptx::umma_commit(&qd_empty[st]);  // Q / dO of this tile: last read by dK / dV
        ATTN_TRACE(true, g, 0);
        if (kDsTmem) {
          if (g >= 1) mma_wait(&dq_free[0], (g - 1) & 1);  // dQ_{g-1} read out of TMEM
        } else if (g >= 2) {
          mma_wait(&dq_free[st], ((g >> 1) & 1) ^ 1);  // dQ_{g-2} drained
        }
        ATTN_TRACE(true, g, 2);
        ptx::tc_fence_after();
#pragma unroll
        for (int k = 0; k < kKV / 16; ++k) {  // dQ = dS K: reduce over 16 keys per step
          if (kDsTmem)  // A = dS from TMEM: 16 keys = 8 columns of bf16 pairs
            ptx::umma_f16_ts(tmem + kDQ, tmem + kDS + k * 8, ptx::smem_desc_sw128(sk + k * 2048, kTileBytes, 1024), id_q,
                             k > 0 ? 1u : 0u);
          else
            ptx::umma_f16(tmem + kDQ + 64 * st,
                          ptx::smem_desc_sw128(sds + (k >> 2) * kTileBytes + (k & 3) * 32, 16, 1024),
                          ptx::smem_desc_sw128(sk + k * 2048, kTileBytes, 1024), id_q, k > 0);
        }
        ptx::umma_commit(mm_done);
        ptx::umma_commit(&dq_full[dq_slot(g)]);
        if (last) ptx::umma_commit(&kv_empty[kvb]);  // this item's K / V no longer read
        q = nx;
      }
    }
  } else if (warp >= 12 && kDqRed) {  // dQ drain warpgroup: vector reductions from registers
    // TMEM -> registers -> red.global.add.v4.f32 straight into the fp32 accumulator: no
    // shared-memory stage (the staged TMA reduce-add moved 64 KB per tile through shared
    // memory, the resource the MMAs' operand reads already nearly saturate)
    const int r = (warp & 3) * 32 + lane;  // TMEM lane: query row
    const uint32_t trow = tmem + (uint32_t((warp & 3) * 32) << 16);
    int g = 0;
    for (BwdSeq q = seq0; q.valid(); ++g) {
      const int b = q.bh / H, hd = q.bh % H, row_base = b * seq, qr = (q.j0 + q.it) * kQ + r;
      ptx::mbar_wait(&dq_full[dq_slot(g)], dq_full_parity(g));
      ptx::tc_fence_after();
      float* dst = dqacc + ((long long)row_base + qr) * (H * kD) + hd * kD;
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t v[32];
        ptx::tmem_ld32(trow + kDQ + 64 * dq_slot(g) + 32 * hh, v);
        ptx::tmem_ld_wait();
        if (hh == 1) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(&dq_free[dq_slot(g)]);
        }
        if (qr < seq) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 32 * hh + 4 * c), "r"(v[4 * c]),
                         "r"(v[4 * c + 1]), "r"(v[4 * c + 2]), "r"(v[4 * c + 3])
                         : "memory");
        }
      }
      q.advance();
    }
  } else if (warp >= 12) {  // dQ drain warpgroup
    const int r = (warp & 3) * 32 + lane;  // TMEM lane: query row
    const int dt = threadIdx.x - 384;
    const uint32_t trow = tmem + (uint32_t((warp & 3) * 32) << 16);
    uint8_t* stage = smem + kB_DQ;  // [2 column halves][128 rows][128 B]
    int g = 0;
    for (BwdSeq q = seq0; q.valid(); ++g) {
      const int b = q.bh / H, hd = q.bh % H, row_base = b * seq, q0 = (q.j0 + q.it) * kQ;
      if (dt == 0) ptx::bulk_wait_read0();  // the previous reduce-adds have read the stage
      ATTN_TRACE(dt == 0, g, 8);
      named_bar_sync(4, 128);
      ptx::mbar_wait(&dq_full[dq_slot(g)], dq_full_parity(g));
      ATTN_TRACE(dt == 0, g, 7);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {  // 32 columns at a time (few registers in this WG)
        uint32_t v[32];
        ptx::tmem_ld32(trow + kDQ + 64 * dq_slot(g) + 32 * hh, v);
        ptx::tmem_ld_wait();
        if (hh == 1) {
          ptx::tc_fence_before();
          ptx::mbar_arrive(&dq_free[dq_slot(g)]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(stage + hh * kTileBytes + r * 128 + ((c ^ (r & 7)) << 4)) =
              make_uint4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
      }
      ptx::fence_proxy_async();
      named_bar_sync(4, 128);
      if (dt == 0) {
        ptx::tma_reduce_add_2d(&tdq, stage, hd * kD, row_base + q0);
        ptx::tma_reduce_add_2d(&tdq, stage + kTileBytes, hd * kD + 32, row_base + q0);
        ptx::bulk_commit();
        ATTN_TRACE(true, g, 9);
      }
      q.advance();
    }
    if (dt == 0) ptx::bulk_wait0();
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kBwdRegsCompute));
    const int g2 = warp >> 2;               // compute warpgroup: key columns [64 g2, 64 g2 + 64)
    const int r = (warp & 3) * 32 + lane;   // TMEM lane: query row (S, dP, dQ) / key row (dK, dV)
    const int ct = threadIdx.x & 127;       // thread within the WG
    const uint32_t trow = tmem + (uint32_t((warp & 3) * 32) << 16);
    const float sl2 = 0.125f * kLog2e;
    uint8_t* sp = smem + kB_P + g2 * kTileBytes;
    uint8_t* sds = smem + kB_DS + g2 * kTileBytes;
    // the WG's P tile doubles as the item epilogue's dK / dV stage; before the next P is
    // written there, the TMA store issued from it must have read it (epi_pending)
    bool epi_pending = false;
    auto stage_release = [&] {
      ptx::fence_proxy_async();
      named_bar_sync(2 + g2, 128);
    };
    // lse and D of this thread's row in tile q (raw; 0 past the sequence / the last tile)
    auto fetch_raw = [&](const BwdSeq& q, float& l, float& d) {
      l = 0.f, d = 0.f;
      if (!q.valid()) return;
      const int qi = (q.j0 + q.it) * kQ + r;
      if (qi < seq) l = lse[(long long)q.bh * seq + qi], d = Dv[(long long)q.bh * seq + qi];
    };
    auto fetch = [&](const BwdSeq& q, float& nl, float& nd) {  // -lse*log2(e), -D of this row
      fetch_raw(q, nl, nd);
      nl = -nl * kLog2e, nd = -nd;
    };
    const float2 sc2 = make_float2(sl2, sl2);
    float nl = 0.f, nd = 0.f;
    if (!lse_bulk) fetch(seq0, nl, nd);
    int g = 0;
    for (BwdSeq q = seq0; q.valid(); ++g) {
      const int b = q.bh / H, hd = q.bh % H, row_base = b * seq;
      const int k0 = q.kb * kKV, q0 = (q.j0 + q.it) * kQ, qr = q0 + r, it = q.it;
      const bool last = it + 1 == q.niter;
      float raw_l = 0.f, raw_d = 0.f;  // (global path) the next tile's lse / D, used after this tile
      if (!lse_bulk) {
        BwdSeq nq = q;
        nq.advance();
        fetch_raw(nq, raw_l, raw_d);
      }
      ATTN_TRACE(threadIdx.x == 0, g, 3);
      ptx::mbar_wait(s_full, g & 1);
      ATTN_TRACE(threadIdx.x == 0, g, 5);
      ptx::tc_fence_after();
      if (lse_bulk) {  // this tile's lse / D landed with its Q / dO (that phase cannot move on
                       // before this tile's ds_full)
        ptx::mbar_wait(&qd_full[g & 1], (g >> 1) & 1);
        const float* ls = reinterpret_cast<const float*>(smem + kB_LSE + (g & 1) * 1024);
        const bool in = qr < seq;
        nl = in ? -ls[r] * kLog2e : 0.f;
        nd = in ? -ls[128 + r] : 0.f;
      }
      uint32_t rs[2][32], rd[2][32];
      ptx::tmem_ld32(trow + kS + 64 * g2, rs[0]);
      ptx::tmem_ld32(trow + kS + 64 * g2 + 32, rs[1]);
      ptx::tmem_ld32(trow + kDP + 64 * g2, rd[0]);
      ptx::tmem_ld32(trow + kDP + 64 * g2 + 32, rd[1]);
      ptx::tmem_ld_wait();
      ATTN_WTRACE(0, g);
      ptx::tc_fence_before();
      ptx::mbar_arrive(st_free);
      // masking only on diagonal / tail tiles (warp-uniform branch): keys of this WG's
      // block at index >= hi drop to a -inf score (P = dS = 0); rows past seq drop out
      if ((CAUSAL && k0 + kKV - 1 > q0) || q0 + kQ > seq || k0 + kKV > seq) {
        const int kg = k0 + 64 * g2;
        const int hi = qr >= seq ? 0 : min(CAUSAL ? qr - kg + 1 : 64, seq - kg);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (32 * h + i >= hi) rs[h][i] = 0xff800000u;
      }
      const float2 nl2 = make_float2(nl, nl), nd2 = make_float2(nd, nd);
      uint32_t pk[32], dk[32];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const int c = 32 * h + i;
          const float2 x = ptx::fma2(make_float2(__uint_as_float(rs[h][i]), __uint_as_float(rs[h][i + 1])), sc2, nl2);
          const float2 p = (kBwdPolyEvery > 0 && (c >> 1) % (kBwdPolyEvery > 0 ? kBwdPolyEvery : 1) == kBwdPolyEvery - 1)
                               ? ptx::ex2_poly2(x)
                               : make_float2(ex2_approx(x.x), ex2_approx(x.y));
          const float2 ds =
              ptx::mul2(p, ptx::add2(make_float2(__uint_as_float(rd[h][i]), __uint_as_float(rd[h][i + 1])), nd2));
          __nv_bfloat162 hp = __floats2bfloat162_rn(p.x, p.y);
          __nv_bfloat162 hs = __floats2bfloat162_rn(ds.x, ds.y);
          pk[c >> 1] = *reinterpret_cast<uint32_t*>(&hp);
          dk[c >> 1] = *reinterpret_cast<uint32_t*>(&hs);
        }
      BwdSeq nx = q;
      nx.advance();
      if (!lse_bulk) nl = -raw_l * kLog2e, nd = -raw_d;  // the next tile's, loaded a tile ago
      ATTN_TRACE(threadIdx.x == 0, g, 11);
      if (g > 0) {  // the previous tile's dV / dK / dQ MMAs have read the P / dS tiles
        ptx::mbar_wait(mm_done, (g - 1) & 1);
        ptx::tc_fence_after();
      }
      ATTN_TRACE(threadIdx.x == 0, g, 10);
      if (epi_pending) {  // the previous item's dK / dV store has read this WG's P tile
        if (ct == 0) ptx::bulk_wait_read0();
        named_bar_sync(2 + g2, 128);
        epi_pending = false;
      }
#pragma unroll
      for (int k8 = 0; k8 < 8; ++k8) {  // 8 keys -> one 16-byte chunk of this WG's block
        const int off = r * 128 + ((k8 ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(sp + off) = make_uint4(pk[4 * k8], pk[4 * k8 + 1], pk[4 * k8 + 2], pk[4 * k8 + 3]);
        *reinterpret_cast<uint4*>(sds + off) = make_uint4(dk[4 * k8], dk[4 * k8 + 1], dk[4 * k8 + 2], dk[4 * k8 + 3]);
      }
      if (kDsTmem) {  // this WG's 64 keys of dS -> TMEM columns [kDS + 32 g2, +32), the dQ MMA's A
        tmem_st32(trow + kDS + 32 * g2, dk);
        tmem_st_wait();
      }
      ATTN_TRACE(threadIdx.x == 0, g, 6);
      ATTN_WTRACE(1, g);
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(ds_full);
      if (last) {  // item epilogue: dK (WG 0, x 1/sqrt(d)) or dV (WG 1)
        ptx::mbar_wait(mm_done, g & 1);
        ptx::tc_fence_after();
        uint32_t v[2][32];
        ptx::tmem_ld32(trow + (g2 == 0 ? kDK : kDV), v[0]);
        ptx::tmem_ld32(trow + (g2 == 0 ? kDK : kDV) + 32, v[1]);
        ptx::tmem_ld_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(acc_free);
        const float sc = g2 == 0 ? 0.125f : 1.f;
        uint4 w[8];  // key row r: 64 bf16 = 8 chunks of 16 bytes
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t w4[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int j = c * 8 + 2 * e;
            __nv_bfloat162 hb = __floats2bfloat162_rn(__uint_as_float(v[j >> 5][j & 31]) * sc,
                                                      __uint_as_float(v[j >> 5][(j & 31) + 1]) * sc);
            w4[e] = *reinterpret_cast<uint32_t*>(&hb);
          }
          w[c] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
        }
        // staged in the swizzled P tile: the TMA store's source and the bias-gradient sums'
#pragma unroll
        for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(sp + r * 128 + ((c ^ (r & 7)) << 4)) = w[c];
        stage_release();
        epi_pending = true;
        if (k0 + kKV <= seq) {  // whole tile inside the sequence: TMA store
          if (ct == 0) {
            ptx::tma_store_2d(&tdqkv, sp, (1 + g2) * H * kD + hd * kD, row_base + k0);
            ptx::bulk_commit();
          }
        } else if (k0 + r < seq) {  // sequence tail: rows past seq belong to the next sequence
          bf16* dst = dqkv + ((long long)row_base + k0 + r) * (3LL * H * kD) + (1 + g2) * (long long)H * kD + hd * kD;
#pragma unroll
          for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(dst + c * 8) = w[c];
        }
        if (dbias) {  // K / V part of the QKV bias gradient: this item's 128 key rows per column
          const int col = ct & 63, r0 = (ct >> 6) * 64;  // keys past seq hold zeros
          float cs = 0.f;
#pragma unroll 8
          for (int rr = r0; rr < r0 + 64; ++rr)
            cs += __bfloat162float(*reinterpret_cast<const bf16*>(sp + rr * 128 + (((col >> 3) ^ (rr & 7)) << 4) +
                                                                 (col & 7) * 2));
          atomicAdd(dbias + (1 + g2) * H * kD + hd * kD + col, cs);
        }
      }
      q = nx;
    }
    if (ct == 0) ptx::bulk_wait0();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
  ATTN_CTA(2);
}

}  // namespace

void attn_fwd_tc(const bf16* qkv, bf16* out, float* lse, int B, int seq, int H, bool causal, cudaStream_t st) {
  const long long ld = 3LL * H * kD;
  const CUtensorMap m = cuda::make_map_2d_bf16(qkv, ld, (long long)B * seq, ld, 64, 128);
  const CUtensorMap mo = cuda::make_map_2d_bf16(out, (long long)H * kD, (long long)B * seq, (long long)H * kD, 64, 128);
  const int items = (seq + kQ - 1) / kQ * B * H;
  const dim3 grid(std::min(items, 2 * cuda::num_sms()));  // persistent: two CTAs per SM
  static bool attr = false;
  if (!attr) {
    CK_CUDA(cudaFuncSetAttribute(k_attn_fwd_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    CK_CUDA(cudaFuncSetAttribute(k_attn_fwd_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    attr = true;
  }
  cuda::launch(causal ? k_attn_fwd_tc<true> : k_attn_fwd_tc<false>, grid, dim3(192), kSmemTotal, st, m, mo, out, lse, seq,
               H, B * H);
  CK_CUDA(cudaGetLastError());
}

// dqkv from dout on the tensor cores; `scratch` as attn_bwd (row dots D, fp32 dQ).
void attn_bwd_tc(const bf16* qkv, const bf16* out, const bf16* dout, const float* lse, bf16* dqkv, float* scratch,
                 int B, int seq, int H, bool causal, cudaStream_t st, float* dbias) {
  if (dbias && (reinterpret_cast<uintptr_t>(dbias) % 16))  // float4 atomics in the dQ pass
    throw chimera::capi::InternalError("attention: the bias-gradient pointer must be 16-byte aligned");
  float* D = scratch;
  float* dq = scratch + attn_dq_offset(B, seq, H);
  const int M = B * seq;
  attn_bwd_dot(out, dout, D, M, seq, H, st, dq);  // + zeroes the dQ accumulator
  const long long ld = 3LL * H * kD;
  const CUtensorMap mq = cuda::make_map_2d_bf16(qkv, ld, (long long)M, ld, 64, 128);
  const CUtensorMap mo = cuda::make_map_2d_bf16(dout, (long long)H * kD, (long long)M, (long long)H * kD, 64, 128);
  const CUtensorMap mdq = cuda::make_map_2d_f32(dq, (long long)H * kD, (long long)M, (long long)H * kD, 32, 128);
  const CUtensorMap mdqkv = cuda::make_map_2d_bf16(dqkv, ld, (long long)M, ld, 64, 128);
  static bool attr = false;
  if (!attr) {
    CK_CUDA(cudaFuncSetAttribute(k_attn_bwd_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem));
    CK_CUDA(cudaFuncSetAttribute(k_attn_bwd_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem));
    attr = true;
  }
  const int items = (seq + kKV - 1) / kKV * B * H;
  const dim3 grid(std::min(items, cuda::num_sms()));  // persistent: one CTA per SM
  cuda::launch(causal ? k_attn_bwd_tc<true> : k_attn_bwd_tc<false>, grid, dim3(kBwdThreads), kBwdSmem, st, mq, mo, mdq,
               mdqkv, lse, D, dqkv, seq, H, B * H, dbias, int(seq % 4 == 0), dq);
  CK_CUDA(cudaGetLastError());
  attn_dq_out(dq, dqkv, M, H, st, dbias);
}

}  // namespace chimera::ops

extern "C" CK_API int ck_attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                                     float* scratch, int B, int seq, int H, int causal, void* st) {
  using chimera::ops::bf16;
  return chimera::capi::guarded([&] {
    chimera::ops::attn_bwd_tc((const bf16*)qkv, (const bf16*)out, (const bf16*)dout, lse, (bf16*)dqkv, scratch, B, seq,
                              H, causal != 0, (cudaStream_t)st, nullptr);
  });
}

extern "C" CK_API int ck_attn_bwd_tc_dbias(const void* qkv, const void* out, const void* dout, const float* lse,
                                           void* dqkv, float* scratch, float* dbias, int B, int seq, int H, int causal,
                                           void* st) {
  using chimera::ops::bf16;
  return chimera::capi::guarded([&] {
    chimera::ops::attn_bwd_tc((const bf16*)qkv, (const bf16*)out, (const bf16*)dout, lse, (bf16*)dqkv, scratch, B, seq,
                              H, causal != 0, (cudaStream_t)st, dbias);
  });
}

extern "C" CK_API int ck_attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int seq, int H, int causal,
                                     void* st) {
  return chimera::capi::guarded([&] {
    chimera::ops::attn_fwd_tc(static_cast<const chimera::ops::bf16*>(qkv), static_cast<chimera::ops::bf16*>(out), lse,
                              B, seq, H, causal != 0, static_cast<cudaStream_t>(st));
  });
}
