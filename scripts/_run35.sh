mkdir -p gpurun_out scripts/_bin
for F in "" "-DCK_GEMM_NOFEED"; do
nvcc -std=c++20 -O3 $F -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2107_06925_b200/csrc/cuda -Ipaper_2107_06925_b200/csrc/host scripts/gemm_trace.cu $(ls build/csrc/*.o | grep -v cuda_gemm) -lcuda -o scripts/_bin/gemm_trace$F > gpurun_out/r02as_build.log 2>&1
for S in "2528 1280 5120" "2528 5120 1280" "2528 3840 1280" "2528 1280 1280"; do
  echo "== $F $S"; CK_GEMM_TILE=pair ./scripts/_bin/gemm_trace$F $S 0 0 0 0 | head -4 | tail -2; CK_GEMM_TILE=pair ./scripts/_bin/gemm_trace$F $S 0 0 0 0 | tail -1
done; done
