// Per-tile mainloop / epilogue timeline of the CTA-pair GEMM for CTA 0.  Build + run:
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr \
//     -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host \
//     scripts/gemm_trace.cu $(ls build/csrc/*.o | grep -v cuda_gemm) -lcuda -o scripts/_bin/gemm_trace
//   scripts/_bin/gemm_trace M N K epi a_mn b_mn
#define CK_GEMM_TRACE 1
#include "../paper_2107_06925_b200/csrc/cuda/gemm.cu"

#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]), epi = atoi(argv[4]);
  const bool a_mn = atoi(argv[5]), b_mn = atoi(argv[6]);
  const int block = argc > 7 ? atoi(argv[7]) : 0;  // CTA to trace
  cudaMemcpyToSymbol(chimera::gemm::g_gemm_trace_block, &block, sizeof(int));
  float* ws = nullptr;  // split-K / stream-K workspace (bf16 epilogues), zero-filled
  const long long ws_elems = 8LL << 20;
  cudaMalloc(&ws, ws_elems * 4);
  cudaMemset(ws, 0, ws_elems * 4);
  __nv_bfloat16 *A, *B, *out, *aux, *out2, *bias;
  cudaMalloc(&A, size_t(M) * K * 2);
  cudaMalloc(&B, size_t(N) * K * 2);
  cudaMalloc(&out, size_t(M) * N * 4);
  cudaMalloc(&aux, size_t(M) * N * 2);
  cudaMalloc(&out2, size_t(M) * N * 2);
  cudaMalloc(&bias, size_t(N) * 2);
  cudaMemset(A, 0, size_t(M) * K * 2);
  cudaMemset(B, 0, size_t(N) * K * 2);
  cudaMemset(aux, 0, size_t(M) * N * 2);
  cudaMemset(bias, 0, size_t(N) * 2);
  chimera::gemm::EpiArgs ep;
  ep.out = out;
  ep.ldo = N;
  ep.bias = (epi == 1 || epi == 2) ? bias : nullptr;
  ep.aux = (epi == 2 || epi == 3) ? aux : nullptr;
  ep.ld_aux = N;
  ep.out2 = epi == 1 ? out2 : nullptr;
  ep.ld_out2 = N;
  ep.ws = ws;
  ep.ws_elems = ws_elems;
  auto run = [&] {
    chimera::gemm::gemm((chimera::gemm::Epi)epi, a_mn, b_mn, M, N, K, A, a_mn ? M : K, B, b_mn ? N : K, ep, 0);
  };
  for (int i = 0; i < 5; ++i) run();
  cudaDeviceSynchronize();
  static long long tr[16][8];
  cudaMemcpyToSymbol(chimera::gemm::g_gemm_trace, tr, sizeof(tr));  // clear stale stamps
  run();
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(tr, chimera::gemm::g_gemm_trace, sizeof(tr));
  const long long c0 = tr[0][0];
  printf("CTA %d: item  mma_start  mma_issued  epi4_start  epi4_end  epi11_start epi11_end  fixup_waited (cycles from item 0 start)\n", block);
  printf("kernel entry -> item0 mma start: %lld cycles\n", tr[0][0] - tr[0][6]);
  for (int t = 0; t < 16 && tr[t][0]; ++t)
    printf("%4d %10lld %11lld %11lld %9lld %11lld %9lld %11lld\n", t, tr[t][0] - c0, tr[t][1] - c0, tr[t][2] - c0,
           tr[t][3] - c0, tr[t][4] - c0, tr[t][5] - c0, tr[t][7] ? tr[t][7] - c0 : -1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 20; ++i) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("avg %.2f us  %.0f TFLOP/s\n", ms * 1000 / 20, 2.0 * M * N * K / (ms / 20 * 1e-3) / 1e12);
  return 0;
}
