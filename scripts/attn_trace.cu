// Phase timeline of the tcgen05 attention forward for CTA 0 plus per-CTA SM/start/end
// stamps.  Build + run (on a B200):
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host \
//     scripts/attn_trace.cu $(ls build/csrc/*.o | grep -v attention_tc) -lcuda -o scripts/_bin/attn_trace
#define CK_ATTN_TRACE 1
#include "../paper_2107_06925_b200/csrc/cuda/attention_tc.cu"

#include <cstdio>
#include <cstdlib>
#include <vector>

// SM clock vs %globaltimer over ~1 ms of spinning: the rate clock64() stamps tick at
__global__ void k_clock_rate(long long* out) {
  long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const long long c0 = clock64();
  do asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  while (t1 - t0 < 1000000);
  out[0] = clock64() - c0, out[1] = t1 - t0;
}

int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 4, seq = argc > 2 ? atoi(argv[2]) : 1024, H = argc > 3 ? atoi(argv[3]) : 16;
  const bool bwd = argc > 4 && argv[4][0] == 'b';
  const int trace_cta = argc > 5 ? atoi(argv[5]) : 0;
  cudaMemcpyToSymbol(chimera::ops::g_attn_trace_cta, &trace_cta, sizeof(int));
  const size_t M = size_t(B) * seq;
  std::vector<__nv_bfloat16> h(M * 3 * H * 64);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = __float2bfloat16(((x >> 8) / 16777216.f - 0.5f) * 2.f);
  }
  __nv_bfloat16 *qkv, *out;
  float* lse;
  cudaMalloc(&qkv, h.size() * 2);
  cudaMalloc(&out, M * H * 64 * 2);
  cudaMalloc(&lse, M * H * 4);
  cudaMemcpy(qkv, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  __nv_bfloat16 *dout, *dqkv;
  float* scratch;
  cudaMalloc(&dout, M * H * 64 * 2);
  cudaMalloc(&dqkv, h.size() * 2);
  cudaMalloc(&scratch, (M * H + M * H * 64) * 4);
  cudaMemcpy(dout, h.data(), M * H * 64 * 2, cudaMemcpyHostToDevice);
  auto run = [&] {
    if (bwd) chimera::ops::attn_bwd_tc(qkv, out, dout, lse, dqkv, scratch, B, seq, H, true, 0);
    else chimera::ops::attn_fwd_tc(qkv, out, lse, B, seq, H, true, 0);
  };
  chimera::ops::attn_fwd_tc(qkv, out, lse, B, seq, H, true, 0);
  for (int i = 0; i < 400; ++i) run();  // clocks up before the traced launch
  long long* clk;
  cudaMalloc(&clk, 16);
  k_clock_rate<<<1, 1>>>(clk);
  run();
  cudaDeviceSynchronize();
  long long clk_h[2];
  cudaMemcpy(clk_h, clk, 16, cudaMemcpyDeviceToHost);
  printf("SM clock during the trace: %.0f MHz (clock64 cycles per us)\n", clk_h[0] * 1e3 / clk_h[1]);
  static long long tr[32][16], cta[4096][3];
  cudaMemcpyFromSymbol(tr, chimera::ops::g_attn_trace, sizeof(tr));
  cudaMemcpyFromSymbol(cta, chimera::ops::g_attn_cta, sizeof(cta));
  const int ncta = std::min((seq + 127) / 128 * B * H, bwd ? 148 : 296);  // persistent grids
  long long t0 = cta[0][1], tend = 0, tmin = cta[0][1];
  for (int i = 0; i < ncta; ++i) tmin = std::min(tmin, cta[i][1]), tend = std::max(tend, cta[i][2]);
  printf("kernel span %.1f us, %d CTAs\n", (tend - tmin) / 1e3, ncta);
  t0 = cta[trace_cta][1];
  printf("CTA%d sm %lld start +%.2f us dur %.2f us\n", trace_cta, cta[trace_cta][0], (t0 - tmin) / 1e3,
         (cta[trace_cta][2] - cta[trace_cta][1]) / 1e3);
  // per-tile stamps relative to kv_full of tile 0 (cycles)
  const long long c0 = bwd ? tr[0][3] : tr[0][1];
  const char* fnames[] = {"tma:k_empty", "mma:k_full", "mma:s_free", "mma:p_full", "sm:wait_s",
                          "sm:s_full",    "sm:ld_done",  "sm:max_done", "sm:o_done", "sm:p_done",
                          "w1:ld_done",   "w2:ld_done",  "w3:ld_done",  "mma:pv_iss"};
  const char* bnames[] = {"mma:dvdk_iss", "mma:ds_full", "mma:dq_free", "c:start", "mma:s_next",
                          "c:s_full",     "c:ds_done",   "dr:dq_full",  "dr:stg_free", "dr:red_iss",
                          "c:mm_done",    "c:math_done", "-"};
  const char** names = bwd ? bnames : fnames;
  printf("%-4s", "j");
  const int nev = bwd ? 13 : 14;
  for (int e = 0; e < nev; ++e) printf(" %12s", names[e]);
  printf("\n");
  for (int j = 0; j < 16; ++j) {
    printf("%-4d", j);
    for (int e = 0; e < nev; ++e) printf(" %12lld", tr[j][e] ? tr[j][e] - c0 : -1);
    printf("\n");
  }
  if (!bwd)
    printf("CTA0 fwd: entry %lld, set-up done %lld, PDL wait done %lld (cycles)\n", tr[0][14] - c0, tr[1][14] - c0,
           tr[2][14] - c0);
  {  // CTA start / end spread
    long long s0 = cta[0][1], s1 = cta[0][1], d0 = cta[0][2] - cta[0][1], d1 = d0;
    for (int i = 0; i < ncta; ++i) {
      s0 = std::min(s0, cta[i][1]), s1 = std::max(s1, cta[i][1]);
      d0 = std::min(d0, cta[i][2] - cta[i][1]), d1 = std::max(d1, cta[i][2] - cta[i][1]);
    }
    printf("CTA starts within %.2f us; CTA durations %.2f .. %.2f us\n", (s1 - s0) / 1e3, d0 / 1e3, d1 / 1e3);
  }
  if (bwd) {  // per compute warp: S/dP loaded, P/dS stored (cycles from the same origin)
    static long long wt[2][32][16];
    cudaMemcpyFromSymbol(wt, chimera::ops::g_attn_warp, sizeof(wt));
    for (int k = 0; k < 2; ++k) {
      printf("%s per warp (w0..w7):\n", k ? "P/dS stored" : "S/dP loaded");
      for (int j = 0; j < 10; ++j) {
        printf("%-4d", j);
        for (int w = 0; w < 8; ++w) printf(" %8lld", wt[k][j][w] - c0);
        printf("\n");
      }
    }
  }
  if (false)
    printf("CTA0 bwd: entry %lld, final drain done %lld, dK/dV stored %lld, bulk wait done %lld, exit %lld (cycles)\n",
           tr[0][13] - c0, tr[0][14] - c0, tr[0][15] - c0, tr[1][13] - c0, tr[1][14] - c0);
  // tail: histogram of CTA end times
  int sm_busy[256] = {0};
  long long last_end[256] = {0};
  for (int i = 0; i < ncta; ++i) {
    sm_busy[cta[i][0]]++;
    last_end[cta[i][0]] = std::max(last_end[cta[i][0]], cta[i][2]);
  }
  long long e_min = tend, e_max = 0;
  for (int s = 0; s < 148; ++s) if (sm_busy[s]) e_min = std::min(e_min, last_end[s]), e_max = std::max(e_max, last_end[s]);
  printf("SM finish spread: first idle SM at %.1f us, last at %.1f us\n", (e_min - tmin) / 1e3, (e_max - tmin) / 1e3);
  if (false) {  // (per-tile-class CTA durations: pre-persistent grids only)
    const int nt = (seq + 127) / 128, BH = B * H;
    for (int c = 0; c < nt; ++c) {
      double sum = 0, mx = 0, first = 1e30, last = 0;
      for (int b = c * BH; b < (c + 1) * BH; ++b) {
        const double d = (cta[b][2] - cta[b][1]) / 1e3;
        sum += d, mx = std::max(mx, d);
        first = std::min(first, (cta[b][1] - tmin) / 1e3), last = std::max(last, (cta[b][2] - tmin) / 1e3);
      }
      printf("grid slice %d: mean %.2f us max %.2f us, starts %.2f us, last end %.2f us\n", c, sum / BH, mx, first,
             last);
    }
  }
  double dur_sum = 0;
  for (int i = 0; i < ncta; ++i) dur_sum += cta[i][2] - cta[i][1];
  printf("mean CTA duration = %.1f us\n", dur_sum / 1e3 / ncta);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 50; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("avg launch %.2f us (traced build)\n", ms * 1000 / 50);
  return 0;
}
